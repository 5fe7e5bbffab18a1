"""Static SASS opcode histogram of one kernel in an object/.so (dev tool).
usage: python tools/sass_hist.py file.o kernel_substring [window]"""
import collections, re, subprocess, sys
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
cur, body = None, []
for line in out.splitlines():
    if "Function :" in line:
        cur = line
        continue
    if cur and sys.argv[2] in cur:
        m = re.search(r"/\*[0-9a-f]{4,6}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m:
            body.append(m.group(2))
c = collections.Counter(body)
print(len(body), "instructions")
print(c.most_common(25))

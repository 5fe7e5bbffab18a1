"""Summarise a RL_GENP_TRACE timeline (tools/run_genp.py on a trace variant):
per super-panel offsets of the lookahead chain's stamps, relative to the lo
stream passing the previous factor_super. usage: python tools/genp_trace_table.py log [every]"""
import sys
lines = [l.split() for l in open(sys.argv[1]) if l.startswith('T ')]
every = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ev = [(int(a[1]), float(a[2])) for a in lines]
call = ev[[i for i, (t, _) in enumerate(ev) if t == 0][-1]:]
t0 = call[0][1]
sp, cur = [], None
for t, x in call:
    if t == 1:
        cur = {1: x}
        sp.append(cur)
    elif cur is not None:
        cur.setdefault(t, x)
names = {2: "u12a", 3: "gA1", 6: "p1", 7: "u12s", 8: "upd", 4: "fs", 5: "gB"}
for i, d in enumerate(sp):
    if i % every and i < len(sp) - 6:
        continue
    s = d[1]
    print(f"{i:2d} {s - t0:8.1f} " + " ".join(f"{v}={d[k] - s:6.1f}" if k in d else f"{v}=  -   " for k, v in names.items()))
print("total", call[-1][1] - t0)

import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, oracle
import paper_1406_5802_b200 as rl
ref = oracle.C.batched_config2(4096, base=7, threads=8, want_lu=True)
out = rl.batched_preprocess_solve_32(ref["a"], ref["g"], ref["b"])
rows = []
for i in range(4096):
    ag = ref["a"][i] @ ref["g"][i]
    k = np.linalg.cond(ag)
    e = np.linalg.norm(out.lu[i] - ref["lu"][i]) / np.linalg.norm(ref["lu"][i])
    ex = np.linalg.norm(out.x[i] - ref["x"][i]) / np.linalg.norm(ref["x"][i])
    mp = np.abs(np.diag(ref["lu"][i])).min()
    # conditioning of leading minors
    km = max(np.linalg.cond(ag[:j, :j]) for j in range(1, 33))
    rows.append((e / k, e, ex, k, km, ref["growth"][i], mp, i))
rows.sort(reverse=True)
for r in rows[:8]: print("scaled %.2e lu %.2e x %.2e kappa %.2e max_minor_kappa %.2e growth %.2e minpiv %.2e i=%d" % r)
print("max lu/(kappa*maxminor)", max(r[1]/(r[3]*r[4]) for r in rows))
print("max x/kappa", max(r[2]/r[3] for r in rows))

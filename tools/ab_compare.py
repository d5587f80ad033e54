"""Compare per-step times of gpurun_out/steps_{A,B,A2}.json (tools/gpu_ab.sh).

    python tools/ab_compare.py [ms|gemm_ms|prep_ms|simt_ms]"""
import json
import sys

fam = sys.argv[1] if len(sys.argv) > 1 else "ms"
import os
keys = [k for k in ("A", "B", "A2", "B2") if os.path.exists(f"gpurun_out/steps_{k}.json")]
L = {k: {r["step"]: r for r in json.load(open(f"gpurun_out/steps_{k}.json"))["steps"]} for k in keys}
A = [k for k in keys if k.startswith("A")]
B = [k for k in keys if k.startswith("B")]
rows = []
for s in L["A"]:
    a = sum(L[k][s][fam] for k in A) / len(A)
    b = sum(L[k][s][fam] for k in B) / len(B)
    if a > 0 or b > 0:
        rows.append((s, a, b))
print("sum over steps: A %.1f  B %.1f ms per slice (%s vs %s)" % (sum(r[1] for r in rows), sum(r[2] for r in rows), A, B))
rows.sort(key=lambda x: -abs(x[2] - x[1]))
print("step   A(avg)  B(avg)   route/shape  (sorted by |B - A|)")
for s, a, b in rows[:30]:
    r = L["A"][s]
    print("%4d %7.2f %7.2f   %s J=%d m=%d n=%d k=%d" % (s, a, b, r["route"], r["J"], r["m"], r["n"], r["k"]))

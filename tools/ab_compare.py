"""Compare per-step times of gpurun_out/steps_{A,B,A2}.json (tools/gpu_ab.sh).

    python tools/ab_compare.py [ms|gemm_ms|prep_ms|simt_ms]"""
import json
import sys

fam = sys.argv[1] if len(sys.argv) > 1 else "ms"
L = {k: {r["step"]: r for r in json.load(open(f"gpurun_out/steps_{k}.json"))["steps"]} for k in ("A", "B", "A2")}
rows = [(s, L["A"][s][fam], L["A2"][s][fam], L["B"][s][fam]) for s in L["A"] if L["A"][s][fam] > 0]
rows.sort(key=lambda x: -abs(x[3] - 0.5 * (x[1] + x[2])))
print("step      A     A2      B   route/shape  (sorted by |B - A|)")
for s, a, a2, b in rows[:30]:
    r = L["A"][s]
    print("%4d %7.2f %7.2f %7.2f   %s J=%d m=%d n=%d k=%d" % (s, a, a2, b, r["route"], r["J"], r["m"], r["n"], r["k"]))
print("sum  %7.1f %7.1f %7.1f" % tuple(sum(r[i] for r in rows) for i in (1, 2, 3)))

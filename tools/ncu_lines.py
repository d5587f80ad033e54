"""Per-source-line summary of an ncu report (--set full --import-source on): the lines with
the most warp-stall samples and shared-memory wavefronts.

    python tools/ncu_lines.py gpurun_out/ncu_x.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ix = {}
for i, k in enumerate(h):
    ix.setdefault(k, i)
lines = []
for r in rows[hi + 1:]:
    if len(r) < len(h) or r[2] != "-":      # source-line rows only (SASS rows carry an address)
        continue
    lines.append(r)


def f(r, k):
    try:
        return float(r[ix[k]])
    except (KeyError, ValueError):
        return 0.0


tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in lines) or 1.0
stall_keys = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
print(f"{'line':>5} {'samp%':>6} {'smem_wf':>9} {'smem_ex':>9} source / top stalls")
for r in sorted(lines, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    s = f(r, "Warp Stall Sampling (All Samples)")
    big = sorted(((k[6:], f(r, k)) for k in stall_keys), key=lambda x: -x[1])[:3]
    print(f"{r[0]:>5} {100 * s / tot:6.1f} {f(r, 'L1 Wavefronts Shared'):9.3g} {f(r, 'L1 Wavefronts Shared Excessive'):9.3g} "
          f"{r[1].strip()[:80]}  {[(k, int(v)) for k, v in big]}")
print("shared wavefronts by line:")
for r in sorted(lines, key=lambda r: -f(r, "L1 Wavefronts Shared"))[:10]:
    print(f"{r[0]:>5} {f(r, 'L1 Wavefronts Shared'):9.3g} ex {f(r, 'L1 Wavefronts Shared Excessive'):9.3g}  {r[1].strip()[:90]}")

# session l: C5 parity (seeded digits); compute-sanitizer memcheck / racecheck / synccheck on small cases
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build_rc=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=900 -p no:cacheprovider -k "c5" -s > gpurun_out/pytest_l.log 2>&1; echo pytest_rc=$?
grep -E "C5 sub|passed|failed|^E  " gpurun_out/pytest_l.log | head
cat > /tmp/sanit.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from tnworkloads import configs
from paper_2310_03978_b200 import Contraction
os.environ.update({"TN_TC_MIN_BIG": "8", "TN_TC_MIN_SMALL": "2", "TN_TC_MIN_K": "2"})
w = configs.small(grid=(3, 4), cycles=8, mode="sparse", n_samples=64, n_slices=4, seed=2)
ref = oracle.contract(w.net, w.path, w.sliced, w.samples)
c = Contraction(device=0, stream=torch.cuda.current_stream())
c.setup(w.net, w.samples, w.path, w.sliced)
c.contract(0, 2); c.contract(2, 4)          # unfused first slice, then fused + graph replay
out = c.sum_slices_host()
A = torch.randn(1, 600, 96, dtype=torch.complex64, device="cuda"); B = torch.randn(1, 40, 96, dtype=torch.complex64, device="cuda")
C = torch.empty(1, 600, 40, dtype=torch.complex64, device="cuda")
c.cgemm(A, B, C, 1, 600, 40, 96)             # narrow, CTA pair
c.close()
print("rel", float(np.linalg.norm(out - ref) / np.linalg.norm(ref)))
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/sanit.py > gpurun_out/sanitizer_$tool.log 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done

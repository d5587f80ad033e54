# short-K promotion interval: A = default (every k-block), B = $KC_ENV (e.g. TN_KCHUNK3_SHORT=2
# TN_SHORTK_MAX=4: every 2 k-blocks for K <= 128); time (A/B step profiles) and error (full-width
# sub-slice parity tests under B)
KC_ENV=${KC_ENV:-"TN_KCHUNK3_SHORT=2"}
AB_ENV_B="$KC_ENV" bash tools/gpu_ab.sh
env $KC_ENV timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout=900 -p no:cacheprovider -s \
    -k "c4_bench or sparse_state or c5_m20" > gpurun_out/pytest_kchunk2.log 2>&1; echo pytest_rc=$?
grep -E "sub-slice|sub-network|passed|failed" gpurun_out/pytest_kchunk2.log | tail -8

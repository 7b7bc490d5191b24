S="tests/test_gpu_2d.py tests/test_gpu_halo.py tests/test_gpu_multirank.py tests/test_gpu_parity.py"
echo "== blocking sequence"; CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest $S -x -q 2>&1 | grep -E "passed|failed|^FAILED|^E  " | head -4
echo "== full suite"; timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "passed|failed|^FAILED|^E  " | head -4
SETS="--prec 64;--prec 32;--prec 64 --order 1;--prec 32 --order 1;--prec 64 --order 0" bash tools/ab_box.sh m6 fm4

# A/B: default build vs tools/variants/$1 (same bench, per-kernel ms)
for lib in default $1; do
  if [ $lib = default ]; then unset HODG_B200_LIB; else export HODG_B200_LIB=tools/variants/$lib/libhodg_b200.so; fi
  timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
  for p in ${PRECS:-64 32}; do echo -n "$lib prec $p: "; timeout 300 python bench.py --steps 20 --warmup 5 --prec $p 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g face %.4f elem %.4f' % (d['value'], d['roofline']['face_ms'], d['roofline']['elem_ms']))"; done
done

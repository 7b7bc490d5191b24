# A/B several variant libs: bash tools/ab_variants.sh "<bench args>" v1 v2 ...
ARGS=$1; shift
for lib in default "$@"; do
  if [ $lib = default ]; then unset HODG_B200_LIB; else export HODG_B200_LIB=tools/variants/$lib/libhodg_b200.so; fi
  echo -n "$lib: "; timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
  echo -n "$lib $ARGS: "; timeout 300 python bench.py --steps 20 --warmup 5 $ARGS 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g face %.4f elem %.4f' % (d['value'], d['roofline']['face_ms'], d['roofline']['elem_ms']))"
done

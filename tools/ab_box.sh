# on the box: parity tests + per-kernel timings for default and variants
# usage: bash tools/ab_box.sh "<bench arg sets separated by ;>" variant...
SETS=${SETS:-"--prec 64;--prec 32"}
for lib in default "$@"; do
  if [ $lib = default ]; then unset HODG_B200_LIB; else export HODG_B200_LIB=tools/variants/$lib/libhodg_b200.so; fi
  echo "== $lib"; timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
  IFS=';' read -ra AR <<< "$SETS"
  for a in "${AR[@]}"; do echo -n "$lib $a: "; timeout 300 python bench.py --no-cpu --no-sub --steps 20 --warmup 5 $a 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g face %.4f elem %.4f' % (d['value'], d['roofline']['face_ms'], d['roofline']['elem_ms']))"; done
done

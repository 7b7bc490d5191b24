python bench.py --no-cpu --no-sub > /dev/null 2>&1
for e in "X=1" "HODG_PDL_MAX_ELEMS=2000000" "HODG_OVERLAP_BND=0" "X=1" "HODG_PDL_MAX_ELEMS=2000000"; do
  for p in 64 32; do echo -n "$e prec $p: "; env $e python bench.py --no-cpu --no-sub --prec $p 2>&1 | grep metric | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g ms/step %.4f' % (d['value'], d['ms_per_step']))"; done
done

python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2 3; do
  for u in 0 2; do
    if [ $u = 0 ]; then unset CG_EW_UNROLL; else export CG_EW_UNROLL=$u; fi
    timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 20 --warmup 5 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('unroll$u', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
  done
done

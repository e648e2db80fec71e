python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/exp_accuracy.py; CG_FAST_EXP=1 python tools/exp_accuracy.py
for i in 1 2 3; do
  timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 20 --warmup 5 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('default', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
  CG_FAST_EXP=1 timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 20 --warmup 5 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('fastexp', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done

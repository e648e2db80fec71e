python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c2 or random or ew or elementwise or c1" > gpurun_out/i32_tests.log 2>&1; echo rc=$? >> gpurun_out/i32_tests.log
for i in 1 2 3; do
  timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 20 --warmup 5 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('idx32', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
  CG_EW_IDX64=1 timeout 300 python bench.py --no-secondary --no-cpu-baseline --steps 20 --warmup 5 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('idx64', round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done > gpurun_out/i32_ab.log 2>&1

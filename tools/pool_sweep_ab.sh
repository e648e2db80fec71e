python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CG_POOL_SWEEP=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "pool or c5 or avg" > gpurun_out/ps_tests.log 2>&1; echo rc=$? >> gpurun_out/ps_tests.log
for i in 1 2; do
  timeout 300 python tools/bench_train.py --configs C5 --iters 5 | grep ms_per | cut -c1-60
  CG_POOL_SWEEP=1 timeout 300 python tools/bench_train.py --configs C5 --iters 5 | grep ms_per | cut -c1-60
done > gpurun_out/ps_bench.log 2>&1
CG_POOL_SWEEP=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:avgpool -c 11 --csv --log-file gpurun_out/ps_launches.csv python tools/bench_train.py --configs C5 --iters 1 > gpurun_out/ncu.log 2>&1

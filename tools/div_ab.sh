./tools/div_check > gpurun_out/div_check.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pool_fusion.py -m gpu -q -x -k "c5 or epilogue or conv or band or rows or c3 or c4" > gpurun_out/div_tests.log 2>&1; echo rc=$? >> gpurun_out/div_tests.log
timeout 400 python tools/bench_train.py --configs C5,C3 --iters 5 > gpurun_out/div_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 130 --csv --log-file gpurun_out/c5_launches_div.csv python tools/bench_train.py --configs C5 --iters 2 > gpurun_out/ncu.log 2>&1

python -c "import __graft_entry__ as g; g.build()" > gpurun_out/t_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_pool_fusion.py tests/test_gpu_fused_coll.py tests/test_gpu_parity.py -m gpu -q -x -k "fusion or c3 or c4 or epilogue or fused" > gpurun_out/t_tests.log 2>&1; echo rc=$? >> gpurun_out/t_tests.log
timeout 300 python tools/bench_train.py --configs C3,C4 --iters 20 > gpurun_out/t_bench.log 2>&1
CG_NO_POOL_FUSION=1 timeout 300 python tools/bench_train.py --configs C3,C4 --iters 20 >> gpurun_out/t_bench.log 2>&1

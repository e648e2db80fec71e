# f2 pooling / conv-epilogue fusion: tests, C4 A/B, launch list
set -x
timeout 600 python -m pytest tests/test_gpu_pool_fusion.py -m gpu -q -x > gpurun_out/r2_pf_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_pf_tests.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c4 or conv" > gpurun_out/r2_pf_parity.log 2>&1; echo rc=$? >> gpurun_out/r2_pf_parity.log
for i in 1 2; do
CG_NO_POOL_FUSION=1 timeout 120 python tools/bench_train.py --configs C4 --iters 20 > gpurun_out/r2_pf_off$i.log 2>&1
timeout 120 python tools/bench_train.py --configs C4 --iters 20 > gpurun_out/r2_pf_on$i.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 140 --csv --log-file gpurun_out/r2_pf_launches.csv python tools/bench_train.py --configs C4 --iters 3 > gpurun_out/ncu.log 2>&1

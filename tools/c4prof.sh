set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "conv_geometries or conv_family or c4_conv" > gpurun_out/r2_bk1.log 2>&1; echo rc=$? >> gpurun_out/r2_bk1.log
timeout 120 python tools/bench_train.py --configs C4 --iters 20 > gpurun_out/r2_bk1_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 100 --csv --log-file gpurun_out/r2_c4_launches4.csv python tools/bench_train.py --configs C4 --iters 3 > gpurun_out/ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$1" -s 2 -c 2 -o gpurun_out/r2_prof -f python tools/bench_train.py --configs C4 --iters 2 > gpurun_out/ncu2.log 2>&1

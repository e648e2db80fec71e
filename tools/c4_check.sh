# C4 conv changes: forced build, parity tests, bench A/B, launch list
python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_03770_b200 import build; build.build(force=True)" > gpurun_out/c4c_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pool_fusion.py -m gpu -q -x -k "c4 or conv or pool" > gpurun_out/c4c_tests.log 2>&1; echo rc=$? >> gpurun_out/c4c_tests.log
timeout 200 python tools/bench_train.py --configs C4 --iters 20 > gpurun_out/c4c_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 140 --csv --log-file gpurun_out/c4c_launches.csv python tools/bench_train.py --configs C4 --iters 3 > gpurun_out/ncu.log 2>&1

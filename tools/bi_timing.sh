CG_EXTRA_NVCC_FLAGS="-DCG_BI_TIMING" python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_03770_b200 import build; build.build(force=True)" > gpurun_out/bi_build.log 2>&1
timeout 200 python tools/bench_train.py --configs C4 --iters 1 > gpurun_out/bi_time.log 2>&1
python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_03770_b200 import build; build.build(force=True)" > gpurun_out/bi_build2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c4 or conv" > gpurun_out/bi_tests.log 2>&1; echo rc=$? >> gpurun_out/bi_tests.log
timeout 200 python tools/bench_train.py --configs C4 --iters 20 > gpurun_out/bi_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 140 --csv --log-file gpurun_out/bi_launches.csv python tools/bench_train.py --configs C4 --iters 3 > gpurun_out/ncu.log 2>&1

CG_EXTRA_NVCC_FLAGS="-DCG_BS_TIMING" python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_03770_b200 import build; build.build(force=True)" > gpurun_out/bs_build.log 2>&1
timeout 200 python tools/bench_train.py --configs C4 --iters 1 > gpurun_out/bs_time.log 2>&1

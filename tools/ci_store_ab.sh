b() { CG_EXTRA_NVCC_FLAGS="$1" python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_03770_b200 import build; build.build(force=True)" > gpurun_out/ci_build.log 2>&1; }
b ""
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pool_fusion.py -m gpu -q -x -k "c4 or conv or pool" > gpurun_out/c4c_tests.log 2>&1; echo rc=$? >> gpurun_out/c4c_tests.log
for c in conv1 conv2; do python tools/conv_iso.py $c; done > gpurun_out/ci_iso.log 2>&1
timeout 200 python tools/bench_train.py --configs C4 --iters 20 >> gpurun_out/ci_iso.log 2>&1
b "-DCG_CI_DIRECT_STORE"
for c in conv1 conv2; do python tools/conv_iso.py $c; done >> gpurun_out/ci_iso.log 2>&1
timeout 200 python tools/bench_train.py --configs C4 --iters 20 >> gpurun_out/ci_iso.log 2>&1

b() { CG_EXTRA_NVCC_FLAGS="$1" python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_03770_b200 import build; build.build(force=True)" > gpurun_out/eg_build.log 2>&1; }
b ""
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pool_fusion.py tests/test_gpu_fused_coll.py -m gpu -q -x -k "dot or tc or conv or c3 or c5 or epilogue or fused or pool" > gpurun_out/eg_tests.log 2>&1; echo rc=$? >> gpurun_out/eg_tests.log
for i in 1 2; do
  b ""; echo "groups=2"; timeout 400 python tools/bench_train.py --configs C5,C3,C4 --iters 5 | grep ms_per | cut -c1-60
  b "-DCG_TC_EPI_GROUPS=1"; echo "groups=1"; timeout 400 python tools/bench_train.py --configs C5,C3,C4 --iters 5 | grep ms_per | cut -c1-60
done > gpurun_out/eg_bench.log 2>&1
b ""

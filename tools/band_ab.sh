b() { CG_EXTRA_NVCC_FLAGS="$1" python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_03770_b200 import build; build.build(force=True)" > gpurun_out/band_build.log 2>&1; }
b ""
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "conv or c5 or band or stem" > gpurun_out/band_tests.log 2>&1; echo rc=$? >> gpurun_out/band_tests.log
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv_band -c 2 --csv --log-file gpurun_out/band_new.csv python tools/bench_train.py --configs C5 --iters 1 > gpurun_out/ncu.log 2>&1
for i in 1 2; do
  b ""; echo new; timeout 300 python tools/bench_train.py --configs C5 --iters 5 | grep ms_per | cut -c1-60
  b "-DCG_SB_BG=2 -DCG_SB_EW=2"; echo old; timeout 300 python tools/bench_train.py --configs C5 --iters 5 | grep ms_per | cut -c1-60
done > gpurun_out/band_bench.log 2>&1
b ""

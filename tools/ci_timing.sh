# conv_img_tc variants (diagnostics); every variant is a forced rebuild
b() { CG_EXTRA_NVCC_FLAGS="$1" python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_03770_b200 import build; build.build(force=True)" > gpurun_out/ci_build.log 2>&1; }
b "-DCG_CI_TIMING -DCG_CI_MMALAT"; timeout 200 python tools/conv_iso.py conv1 3 > gpurun_out/ci_time.log 2>&1; timeout 200 python tools/conv_iso.py conv2 3 >> gpurun_out/ci_time.log 2>&1

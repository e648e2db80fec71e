b() { CG_EXTRA_NVCC_FLAGS="$1" python -c "
import sys; sys.path.insert(0,'.')
from paper_1812_03770_b200 import build; build.build()" > gpurun_out/ci_build.log 2>&1; }
for v in "" "-DCG_CI_DIRECT_STORE"; do
  b "$v"; echo "== build [$v]"
  for c in conv1 conv2; do
    python tools/conv_iso.py $c; CG_NO_POOL_FUSION=1 python tools/conv_iso.py $c
  done
  timeout 200 python tools/bench_train.py --configs C4 --iters 20 | tail -1 | cut -c1-70
done

cd $GRAFT_REPO_ROOT
CG_EXTRA_NVCC_FLAGS=-DCG_SB_TIMING python -c "from paper_1812_03770_b200 import build; build.build(force=True)" > gpurun_out/bt_build.log 2>&1
timeout 200 python tools/c5_quick.py 256 > gpurun_out/band_time.log 2>&1
python -c "from paper_1812_03770_b200 import build; build.build(force=True)" > gpurun_out/bt_build2.log 2>&1

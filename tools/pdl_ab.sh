# PDL: GPU suite, then C1/C3/C4/C5 with and without the attribute (interleaved)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pdl_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pdl_gpu.log 2>&1; echo rc=$? >> gpurun_out/pdl_gpu.log
for i in 1 2; do
  timeout 400 python tools/bench_train.py --configs C3,C4,C5 --iters 20 > gpurun_out/pdl_on$i.log 2>&1
  CG_NO_PDL=1 timeout 400 python tools/bench_train.py --configs C3,C4,C5 --iters 20 > gpurun_out/pdl_off$i.log 2>&1
done

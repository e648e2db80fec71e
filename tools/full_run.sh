python -c "import __graft_entry__ as g; g.build()" > gpurun_out/full_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/full_gpu.log 2>&1; echo rc=$? >> gpurun_out/full_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/full_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/full_bench.log 2>&1

#!/bin/bash
# GPU parity pass: build, then the -m gpu tests (optionally a -k filter), each bounded by timeout.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { cat gpurun_out/build.log; exit 1; }
timeout ${T:-900} python -m pytest tests -m gpu -q -x ${K:+-k "$K"} > gpurun_out/pytest_gpu.log 2>&1; rc=$?
tail -40 gpurun_out/pytest_gpu.log
exit $rc

#!/bin/bash
# C2 fused-kernel sweep: rows in flight per thread (CG_EW_UNROLL) x blocks/SM cap.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()"
for U in ${US:-1 2 4}; do for B in ${BS:-0}; do for rep in 1 2; do
  v=$(CG_EW_UNROLL=$U CG_EW_BLOCKS_PER_SM=$B timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])")
  echo "U=$U blocks_cap=$B -> $v"
done; done; done

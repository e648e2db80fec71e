#!/bin/bash
# A/B of the software-pipelined row-mode EW kernel on C2 (same box, interleaved runs).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()"
for rep in 1 2 3; do for P in 0 1; do
  v=$(CG_EW_PREFETCH=$P timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])")
  echo "prefetch=$P -> $v"
done; done

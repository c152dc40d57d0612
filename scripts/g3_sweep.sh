#!/bin/bash
# developer loop: build the library with each flag set and time the default counting kernel on cfg3 / cfg4
# usage: scripts/g3_sweep.sh "<flags A>" "<flags B>" ...   (run locally; each variant is one gpurun call)
i=0
for flags in "$@"; do
  i=$((i+1))
  WFCU_NVCC_EXTRA="$flags" python -m paper_2206_05269_b200.build --force > /dev/null || exit 1
  /usr/local/graft/bin/gpurun --timeout 600 -- "for r in 1 2; do python scripts/quick_bench.py 954 50000 2>&1 | grep median; done; python scripts/quick_bench.py 954 1000000 2>&1 | grep median" > gpurun_out/g3_sweep_$i.log 2>&1
  echo "== [$flags]"; grep median gpurun_out/g3_sweep_$i.log
done

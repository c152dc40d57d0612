#!/bin/bash
# developer sweep (GPU box): keys per warp tile of the dense radix passes of the sort + RLE counting path
for t in "$@"; do
  export WFCU_NVCC_EXTRA="-DWFCU_DENSE_TILE=$t"
  python -m paper_2206_05269_b200.build --force > /dev/null 2>&1 || { echo "tile $t: build failed"; continue; }
  echo "tile $t: $(timeout 200 python scripts/tokenize_probe.py ${DOCS:-954} 2>&1 | tail -1)"
done
unset WFCU_NVCC_EXTRA
python -m paper_2206_05269_b200.build --force > /dev/null 2>&1

#!/bin/bash
# developer sweep (GPU box): build variants of sanitize.cu and time them
for flags in "$@"; do
  export WFCU_NVCC_EXTRA="$flags"
  python -m paper_2206_05269_b200.build --force > /dev/null 2>&1 || { echo "[$flags]: build failed"; continue; }
  echo "[$flags]"; timeout 200 python scripts/sanitize_probe.py 2>&1 | tail -3
done
unset WFCU_NVCC_EXTRA
python -m paper_2206_05269_b200.build --force > /dev/null 2>&1

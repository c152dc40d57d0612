#!/bin/bash
# developer sweep (GPU box): sweep_flags.sh "<command>" "<nvcc flags 1>" "<nvcc flags 2>" ...
cmd="$1"; shift
for flags in "$@"; do
  export WFCU_NVCC_EXTRA="$flags"
  python -m paper_2206_05269_b200.build --force > /dev/null 2>&1 || { echo "[$flags]: build failed"; continue; }
  echo "[$flags] $(bash -c "$cmd" 2>&1 | tail -1)"
done
unset WFCU_NVCC_EXTRA
python -m paper_2206_05269_b200.build --force > /dev/null 2>&1

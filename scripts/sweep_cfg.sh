#!/bin/bash
# developer sweep of the counting kernel's launch shape (run on the GPU box): "warps sets medslots"
for cfg in "${@:-28 3840 256}"; do
  set -- $cfg
  export WFCU_NVCC_EXTRA="-DWFCU_COUNT_WARPS=$1 -DWFCU_COUNT_SETS=$2 -DWFCU_COUNT_MED_SLOTS=$3"
  python -m paper_2206_05269_b200.build --force > /dev/null 2>&1 || { echo "cfg $cfg: build failed"; continue; }
  echo "cfg warps=$1 sets=$2 med=$3: $(timeout 100 python scripts/quick_bench.py ${DOCS:-954} ${VOCAB:-50000} 2>&1 | grep 'wordcount median')"
done
unset WFCU_NVCC_EXTRA
python -m paper_2206_05269_b200.build --force > /dev/null 2>&1

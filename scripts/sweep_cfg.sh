#!/bin/bash
# developer sweep of the fast kernel's launch shape (run on the GPU box)
for cfg in "24 8192 1024" "28 8192 512" "32 4096 1024" "32 4096 512" "16 8192 1024" "20 8192 1024"; do
  set -- $cfg
  export WFCU_NVCC_EXTRA="-DWFCU_FAST_WARPS=$1 -DWFCU_FAST_SLOTS=$2 -DWFCU_FAST_MED_SLOTS=$3"
  python -m paper_2206_05269_b200.build --force > /dev/null 2>&1 || { echo "cfg $cfg: build failed"; continue; }
  echo "cfg warps=$1 slots=$2 med=$3: $(timeout 100 python scripts/quick_bench.py ${DOCS:-954} ${VOCAB:-50000} 2>&1 | grep 'wordcount median')"
done
unset WFCU_NVCC_EXTRA
python -m paper_2206_05269_b200.build --force > /dev/null 2>&1

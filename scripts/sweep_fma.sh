#!/bin/bash
# developer sweep (run on the GPU box): which range-test additions of classify4 go to the FMA pipe (WFCU_FMA_ADDS bit mask)
for m in "${@:-0}"; do
  export WFCU_NVCC_EXTRA="-DWFCU_FMA_ADDS=$m"
  python -m paper_2206_05269_b200.build --force > /dev/null 2>&1 || { echo "mask $m: build failed"; continue; }
  echo "mask $m: $(timeout 100 python scripts/quick_bench.py ${DOCS:-954} ${VOCAB:-50000} 2>&1 | grep 'wordcount median')"
done
unset WFCU_NVCC_EXTRA
python -m paper_2206_05269_b200.build --force > /dev/null 2>&1

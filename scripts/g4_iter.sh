#!/bin/bash
# developer loop: build with extra nvcc flags, time the count kernel on cfg3 and capture one ncu profile
# usage: scripts/g4_iter.sh <tag> [extra nvcc flags...]
tag=$1; shift
WFCU_NVCC_EXTRA="$*" python -m paper_2206_05269_b200.build --force > /dev/null || exit 1
/usr/local/graft/bin/gpurun --timeout 600 -- "WFCU_COUNT_VARIANT=0 python scripts/quick_bench.py 954 50000 2>&1 | head -4 > gpurun_out/${tag}_qb.log; WFCU_COUNT_VARIANT=0 ncu --set full --clock-control none --import-source on -k regex:wc_count -s 3 -c 1 -o gpurun_out/${tag} python scripts/prof_wc.py 954 50000 > gpurun_out/${tag}_ncu.log 2>&1" > gpurun_out/${tag}_call.log 2>&1
tail -2 gpurun_out/${tag}_call.log | head -1
grep -E "median|stats" gpurun_out/${tag}_qb.log
python scripts/ncu_summary.py gpurun_out/${tag}.ncu-rep 976897 2>&1 | grep -E "time_duration|registers|inst_executed.sum|issue_active|wavefronts_mem_shared|bank_conflicts" 
python scripts/ncu_summary.py gpurun_out/${tag}.ncu-rep 976897 2>&1 | sed -n '/stall samples/,/code regions/p' | head -8

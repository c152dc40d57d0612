#!/bin/bash
# Round-end evidence in one GPU call: full GPU suite, smoke, both bench arms, the other workloads, the ncu launch list
# of the bench command and one full capture of the counting kernel (summarised on the box: the .ncu-rep is too large to
# travel).  Run on the GPU box: /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash scripts/final_pass.sh'
out=gpurun_out/final
mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > $out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.txt 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_reference.json 2> $out/bench_reference.err
python bench.py --steps 20 --warmup 3 > $out/bench.json 2> $out/bench.err
python bench.py --workload cfg4 --docs 954 --steps 20 --warmup 3 > $out/bench_cfg4.json 2> /dev/null
python bench.py --workload cfg5 --steps 5 --warmup 3 > $out/bench_cfg5.json 2> /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-mapreduce --e2e-steps 1 > $out/bench_under_ncu.log 2>&1
WFCU_COUNT_VARIANT=0 ncu --set full --clock-control none --import-source on -k regex:wc_count -s 3 -c 1 -o /tmp/final_cfg3 python scripts/prof_wc.py 954 50000 > $out/ncu_cfg3.log 2>&1
python scripts/ncu_summary.py /tmp/final_cfg3.ncu-rep 976897 > $out/wc_count_cfg3_summary.txt 2>&1
python scripts/ncu_smem.py /tmp/final_cfg3.ncu-rep > $out/wc_count_cfg3_smem.txt 2>&1
python scripts/ncu_mix.py /tmp/final_cfg3.ncu-rep > $out/wc_count_cfg3_mix.txt 2>&1
tail -2 $out/pytest_gpu.txt; cat $out/smoke.txt | tail -1
python - <<'PY'
import json
for f in ("bench_reference", "bench", "bench_cfg4", "bench_cfg5"):
    try:
        d = json.loads(open(f"gpurun_out/final/{f}.json").read().strip().splitlines()[-1])
        print(f, d.get("value"), (d.get("roofline") or {}).get("frac"), (d.get("e2e") or {}).get("value"), d.get("gpu_launches"), (d.get("parity") or {}).get("equal"))
    except Exception as e:
        print(f, "unreadable:", e)
PY
head -12 $out/wc_count_cfg3_summary.txt

"""Summarise an .ncu-rep (read here, no GPU): key metrics, stall reasons, hot code regions."""
import csv, subprocess, sys, io
rep = sys.argv[1]
rows_hint = float(sys.argv[2]) if len(sys.argv) > 2 else None   # number of 512-byte rows, for per-row counts
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'launch__shared_mem_per_block_dynamic',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'lts__t_sector_hit_rate.pct', 'sm__cycles_elapsed.max',
        'smsp__inst_executed_op_shared_atom.sum', 'smsp__inst_executed_op_global_atom.sum', 'smsp__inst_executed_op_global_red.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'sm__inst_executed_pipe_lsu.sum', 'sm__inst_executed_pipe_alu.sum', 'sm__inst_executed_pipe_fma.sum']
print("== metrics ==")
for h, u, v in zip(hdr, units, vals):
    if h in want:
        print(f"{h:72s} {v:>18s} {u}")
print("== stall samples ==")
st = [(h, int(float(v))) for h, v in zip(hdr, vals) if 'pcsamp_warps_issue_stalled' in h and 'not_issued' not in h]
tot = sum(v for _, v in st) or 1
for h, v in sorted(st, key=lambda x: -x[1])[:10]:
    print(f"{h.split('stalled_')[1]:28s} {v:8d} {100*v/tot:5.1f}%")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]; data = rows[2:]
ia, isamp, isrc, iaddr = hdr.index("Instructions Executed"), hdr.index("# Samples"), hdr.index("Source"), hdr.index("Address")
base = int(data[0][iaddr], 16)
tot_i = sum(int(r[ia]) for r in data)
print(f"== code regions (total {tot_i/1e6:.1f}M warp-instructions" + (f", {tot_i/rows_hint:.0f} per row" if rows_hint else "") + ") ==")
seg = []; cur = None
for r in data:
    c = int(r[ia])
    if cur and abs(c - cur['cnt']) <= 0.03 * max(cur['cnt'], 1):
        cur['n'] += 1; cur['inst'] += c; cur['samp'] += int(r[isamp]); cur['end'] = int(r[iaddr], 16) - base
    else:
        cur = {'start': int(r[iaddr], 16) - base, 'end': int(r[iaddr], 16) - base, 'cnt': c, 'n': 1, 'inst': c, 'samp': int(r[isamp]), 'first': r[isrc].strip()}
        seg.append(cur)
for s in seg:
    if s['inst'] > 0.004 * tot_i or s['samp'] > 0.01 * tot:
        per = f"{s['cnt']/rows_hint:6.2f}/row" if rows_hint else ""
        print(f"{s['start']:5x}-{s['end']:5x} n={s['n']:3d} cnt={s['cnt']:>9d} {per} inst={s['inst']/1e6:7.2f}M samp={s['samp']:6d}  {s['first'][:50]}")
if "--dump" in sys.argv:
    iavg = hdr.index("Avg. Threads Executed")
    for r in data:
        print(f"{int(r[iaddr],16)-base:5x} {int(r[ia]):>9d} {int(r[isamp]):>6d} {float(r[iavg]):5.1f}  {r[isrc].strip()[:90]}")

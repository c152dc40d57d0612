#!/usr/bin/env python
"""bench.py -- the headline benchmark of the word-frequency hot path on B200.

    python bench.py --gpus N --steps K --warmup W [--impl reference] [--workload cfg3|cfg4|cfg5]

metric   word-count corpus GB/s (BASELINE.json): bytes of corpus counted per second,
         whole job over all N GPUs, GB = 1e9 bytes.
workload cfg3 (default): synthetic Zipf(s=1.1) corpus, 50k-word vocabulary, 954 one-MiB
         documents (1.0003 GB) PER GPU, documents assigned round-robin (d mod N); at
         N > 1 every step ends with the hash-partitioned all-to-all merge.  Weak scaling.
         cfg4: 32 GB total, 1M-word vocabulary, document-sharded over N >= 2 GPUs.
         cfg5: four speaker corpora (1 GB each, 1 M-word vocabulary, 1 % speaker-specific words), N = 1:
         a step counts the four corpora, pools the other three per speaker (device merges) and produces
         the per-speaker top-25 and 25 most distinctive words (proj/src/cli.cpp:176-230) on the device.
step     reset the count table + one pass of the fused tokenizer/count kernels over the
         rank's resident shard (+ partition / all-to-all / merge-insert at N > 1).
value    inputs resident in HBM, CUDA-event timed, max over ranks.
e2e      the same step through the host-buffer C-ABI call (wfcu_counter_count_host:
         pack -> pinned staging -> H2D -> count) plus the export of the ordered table to
         host memory; wall clock around synchronised steps, max over ranks.
The reference arm (--impl reference) times the UNMODIFIED reference's run_wordcount
(oracle/_ref, all host threads) on a bounded sample of the same corpus.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DOC_BYTES = 1 << 20
SEED = 1
ZIPF_S = 1.1
WORKLOADS = {
    # name: (vocab, docs per GPU (None = total/N), total docs (None = per-GPU * N), scaling)
    "cfg3": dict(vocab=50000, docs_per_gpu=954, total_docs=None, scaling="weak",
                 name="word count, synthetic Zipf(1.1) corpus, 50k vocabulary, 1 GB per GPU"),
    "cfg4": dict(vocab=1000000, docs_per_gpu=None, total_docs=30518, scaling="strong",
                 name="word count, synthetic Zipf(1.1) corpus, 1M vocabulary, 32 GB document-sharded"),
}
METRIC = "wordcount_corpus_GBps"
UNIT = "GB/s"


def ncu_traffic(kernel: str, nbytes: int, vocab: int):
    """dram__bytes_read + dram__bytes_write of one launch, from the committed ncu capture of this config
    (same kernel, same shard size, same vocabulary), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            entries = json.load(f)
        for name, t in entries.items():
            if name.split(":")[0] == kernel and t["bytes_per_gpu"] == nbytes and t.get("vocab") == vocab:
                return t["dram_bytes_read"] + t["dram_bytes_write"]
    except Exception:
        pass
    return None


def measured_peak_gbs():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clock and throttle reasons sampled through NVML DURING the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[int, int]] = []
        self.max_mhz = None
        self.stop = threading.Event()
        self.thread = None
        self.error = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            visible = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = self.index
            if visible:
                try:
                    idx = int(visible.split(",")[self.index])
                except (ValueError, IndexError):
                    pass
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except Exception as e:   # no NVML: report it, never fake a reading
            self.error = repr(e)
        return self

    def _pump(self):
        n = self.nvml
        while not self.stop.is_set():
            try:
                mhz = n.nvmlDeviceGetClockInfo(self.handle, n.NVML_CLOCK_SM)
                try:
                    reasons = n.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                except Exception:
                    reasons = n.nvmlDeviceGetCurrentClocksThrottleReasons(self.handle)
                self.samples.append((mhz, reasons))
            except Exception as e:
                self.error = repr(e)
                return
            time.sleep(0.001)

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "error": self.error}
        n = self.nvml
        names = {"hw_slowdown": getattr(n, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
                 "hw_thermal_slowdown": getattr(n, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
                 "sw_thermal_slowdown": getattr(n, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
                 "sw_power_cap": getattr(n, "nvmlClocksThrottleReasonSwPowerCap", 0x4)}
        mhz = sorted(m for m, _ in self.samples)
        seen = 0
        for _, r in self.samples:
            seen |= r
        return {"sm_mhz": mhz[len(mhz) // 2], "sm_max_mhz": self.max_mhz,
                "reasons": sorted(k for k, bit in names.items() if seen & bit), "samples": len(mhz)}


def bind_to_gpu_numa_node(torch, index: int) -> dict:
    """Pinned host buffers should live on the NUMA node the GPU hangs off, or PCIe reads cross the
    socket interconnect.  Bind this process to that node's cores before any host allocation
    (first-touch places the pages); returns what was done for the JSON line."""
    info = {"node": None, "cpus": None}
    try:
        p = torch.cuda.get_device_properties(index)
        bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/numa_node") as f:
            node = int(f.read().strip())
        if node < 0:
            return info
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            spec = f.read().strip()
        cpus = set()
        for part in spec.split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        allowed = os.sched_getaffinity(0)
        use = cpus & allowed
        if use:
            os.sched_setaffinity(0, use)
            info = {"node": node, "cpus": len(use)}
    except Exception:
        pass
    return info


def plan(workload: str, world: int, rank: int, docs_override: int | None):
    w = WORKLOADS[workload]
    if w["total_docs"] is None:
        per = docs_override or w["docs_per_gpu"]
        total = per * world
    else:
        total = docs_override or w["total_docs"]
    my_docs = list(range(rank, total, world))   # the reference's rule: document d -> worker d mod n
    return w, total, my_docs


def build_corpus(capi, np, torch, vocab: int, docs: list[int], stride: int):
    """The rank's shard as one pinned host buffer: documents docs[0], docs[0]+stride, ..."""
    n = len(docs) * DOC_BYTES
    host = torch.empty(max(n, 16), dtype=torch.uint8).pin_memory()
    arr = host.numpy()
    if docs:
        capi.synth_corpus_strided(SEED, docs[0], stride, len(docs), vocab, ZIPF_S, 0, DOC_BYTES, out=arr)
    return host, n


def run_reference(args) -> None:
    """The reference's own CPU implementation (wfc::run_wordcount, unmodified sources compiled into oracle/_ref) on
    this box's host cores, on the b200 arm's config: every step counts the WHOLE shard of one GPU.  The corpus comes
    from the stand-alone generator (oracle/libwfsynth.so): the CUDA library is never mapped into this process."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import oracle
    oracle.build()
    cores = os.cpu_count() or 1
    w, total, my_docs = plan(args.workload, max(args.gpus, 1), 0, args.docs)
    use_ref = oracle.ref_available()
    cpu = oracle.ref() if use_ref else oracle.port()
    k = len(my_docs)
    same_config = True
    if args.sample_docs:
        k, same_config = min(k, args.sample_docs), args.sample_docs >= k
    else:
        # run_wordcount keeps every token as a std::string (a few tens of bytes of host memory per corpus byte at its
        # peak): bound the shard by what the box has, and say so
        try:
            import psutil
            fit = int(psutil.virtual_memory().available * 0.6 / (40 * DOC_BYTES))
            if fit < k:
                k, same_config = max(8, fit), False
        except Exception:
            pass
    blob = oracle.synth_corpus(SEED, my_docs[0], k, w["vocab"], ZIPF_S, 0, DOC_BYTES, doc_stride=max(args.gpus, 1))
    docs = [blob[i * DOC_BYTES:(i + 1) * DOC_BYTES] for i in range(k)]

    def one():
        t0 = time.perf_counter()
        if use_ref:
            table, _ = cpu.run_wordcount(docs, cores)
        else:
            table = cpu.wordcount(docs)
        return time.perf_counter() - t0, len(table)

    for _ in range(args.warmup):
        one()
    t0 = time.perf_counter()
    distinct = 0
    for _ in range(args.steps):
        _, distinct = one()
    dt = time.perf_counter() - t0
    nbytes = k * DOC_BYTES
    value = nbytes * args.steps / dt / 1e9
    sample = (f"{k} of the {len(my_docs)} one-MiB documents of one GPU's shard ({nbytes / 1e6:.0f} MB) per step, "
              f"{'wfc::run_wordcount(corpus, n_workers=%d)' % cores if use_ref else 'oracle port, serial'}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": w["scaling"],
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": w["name"], "vocab": w["vocab"], "zipf_s": ZIPF_S, "doc_bytes": DOC_BYTES, "seed": SEED,
                   "documents": total, "bytes_per_step": nbytes, "same_config": same_config,
                   "sample": sample, "distinct_words": distinct},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores if use_ref else 1,
                         "kind": "reference" if use_ref else "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(capi, vocab: int, total_docs: int):
    """The reference CPU path on this box's host cores, bounded sample (rank 0, N=1 only).
    Returns (the JSON object, documents in the sample, the reference's table of the sample)."""
    import oracle
    cores = os.cpu_count() or 1
    use_ref = oracle.ref_available()
    cpu = oracle.ref() if use_ref else oracle.port()
    k, cap = 8, 256   # run_wordcount keeps every token as a std::string: bound the sample
    blob = capi.synth_corpus(SEED, 0, cap, vocab, ZIPF_S, 0, DOC_BYTES)
    docs = [blob[i * DOC_BYTES:(i + 1) * DOC_BYTES] for i in range(cap)]

    def one(d):
        t0 = time.perf_counter()
        table = cpu.run_wordcount(d, cores)[0] if use_ref else cpu.wordcount(d)
        return time.perf_counter() - t0, table
    t, table = one(docs[:k])
    if t < 5.0:      # grow the sample towards ~10-20 s of CPU work, at most 256 documents
        k = int(min(cap, max(k, k * 12.0 / max(t, 1e-3))))
        t, table = one(docs[:k])
    nbytes = k * DOC_BYTES
    return {"value": nbytes / t / 1e9, "unit": UNIT, "cores": cores if use_ref else 1,
            "kind": "reference" if use_ref else "port",
            "sample": f"first {k} of {total_docs} one-MiB documents ({nbytes / 1e6:.0f} MB), one run of "
                      f"{'wfc::run_wordcount with n_workers=%d' % cores if use_ref else 'the serial oracle port'}, {t:.1f} s"}, k, table


def parity_check(capi, dev_ptr: int, k: int, slots: int, ref_table: dict) -> dict:
    """The table the timed kernels build, checked against the reference's: the first k documents of the resident
    shard are counted once more into a fresh counter and the exported (ordered) table is compared entry by entry."""
    c = capi.Counter(table_slots=slots)
    c.count_dev(dev_ptr, k * DOC_BYTES)
    blob, lens, counts = c.export()
    words = capi.unpack_words(blob, lens)
    want = sorted(ref_table.items())
    equal = len(words) == len(want) and all(a == b[0] and int(n) == b[1] for a, n, b in zip(words, counts.tolist(), want))
    return {"checked": True, "docs": k, "bytes": k * DOC_BYTES, "distinct": len(words), "equal": bool(equal),
            "against": "reference run_wordcount table of the same documents (std::map order, exact counts)"}


def run_b200(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2206_05269_b200 import capi
    from paper_2206_05269_b200.exchange import AsyncExchange, DeviceOps, ExchangeOverflow, hash_partition_merge

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.backend == "gloo":
        local_rank = local_rank % max(torch.cuda.device_count(), 1)
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: the product has no CPU path")
    torch.cuda.set_device(local_rank)
    device = torch.device("cuda", local_rank)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:   # gloo carries CUDA tensors through the host: lets 2 ranks share one GPU in tests
            dist.init_process_group("gloo")
    if world != max(args.gpus, 1):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    all_cpus = os.sched_getaffinity(0)
    numa = bind_to_gpu_numa_node(torch, local_rank)
    w, total_docs, my_docs = plan(args.workload, world, rank, args.docs)
    host, nbytes = build_corpus(capi, np, torch, w["vocab"], my_docs, world)
    dev = host.to(device, non_blocking=True)
    torch.cuda.synchronize()
    slots = 1 << 20 if w["vocab"] <= 100000 else 1 << 22
    local = capi.Counter(table_slots=slots)
    owned = capi.Counter(table_slots=slots) if world > 1 else None
    ops = DeviceOps(torch, device)
    stream = torch.cuda.current_stream(device).cuda_stream

    # N > 1: the merge runs without a host synchronisation per step (fixed-capacity regions, sizes read
    # on the device); its sticky overflow / long-token flags are read once, inside the timed region,
    # after the K steps -- if they are raised the run is repeated with the synchronising merge.
    # By default the all-to-all and the merge of step k run on a second stream under the count of step k+1 (two owned
    # tables alternate; --no-overlap-exchange keeps everything on one stream).
    overlap = world > 1 and not args.sync_exchange and not args.no_overlap_exchange
    ax = AsyncExchange(local, ops, dist, entries_hint=w["vocab"], overlap=overlap) if world > 1 and not args.sync_exchange else None
    owned_pair = [owned, capi.Counter(table_slots=slots)] if overlap else [owned]
    last_owned = [owned]

    def step():
        local.reset(stream)
        local.count_dev(dev.data_ptr(), nbytes, stream)
        if world > 1:
            if ax is not None:
                o = owned_pair[ax.steps % len(owned_pair)]
                ax.slot_ready()          # overlap: the merge that last used this table has run (an event, no host wait)
                o.reset(stream)
                ax.step(local, o)
                last_owned[0] = o
            else:
                owned.reset(stream)
                hash_partition_merge(local, owned, ops, dist)
                last_owned[0] = owned

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    local.status(stream)
    if ax is not None:
        try:
            ax.finish()
        except ExchangeOverflow as e:      # collective decision: the flags were all-reduced
            if rank == 0:
                print(f"warning: {e}; using the synchronising merge", file=sys.stderr)
            ax = None
            step()
            barrier()

    # ---- resident-data timing: exactly K steps, CUDA events, max over ranks --------------------
    launches0 = capi.launch_count()
    local.set_timing(True)
    local.take_kernel_ms()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        barrier()
        e0.record()
        for _ in range(args.steps):
            step()
        if ax is not None:
            ax.finish()     # raises if a step left anything behind (none did in the warm-up)
        e1.record()
        barrier()
    total_ms = e0.elapsed_time(e1)
    kernel_ms, kernel_launches = local.take_kernel_ms()
    local.set_timing(False)
    launches = capi.launch_count() - launches0
    t = torch.tensor([total_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    table = last_owned[0] if world > 1 else local
    table.status(stream)
    distinct, tokens, _ = table.stats(stream)
    all_bytes = torch.tensor([nbytes, distinct, tokens], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(all_bytes)
    job_bytes, job_distinct, job_tokens = (int(v) for v in all_bytes.tolist())
    ms_per_step = total_ms / args.steps
    value = job_bytes / (ms_per_step * 1e-3) / 1e9

    # ---- end to end through the host-buffer call (pinned staging, H2D, count, export D2H) ------
    arr = host.numpy()
    docs = capi.HostDocs([arr[i * DOC_BYTES:(i + 1) * DOC_BYTES] for i in range(len(my_docs))])   # pointer/length arrays, built once
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    d2h = 0
    result = None      # page-locked result arrays, allocated once by the caller and reused (the C ABI fills caller buffers)

    def pinned_array(dtype, n):
        return torch.empty(n * np.dtype(dtype).itemsize, dtype=torch.uint8).pin_memory().numpy().view(dtype)

    def e2e_step():
        nonlocal d2h, result
        local.reset()
        local.count_host(docs)
        if world > 1:
            owned.reset(stream)
            hash_partition_merge(local, owned, ops, dist)     # the synchronising form: one-shot use
            torch.cuda.synchronize()
        table = owned if world > 1 else local
        if result is None:
            rows, _, key_bytes = table.stats()
            result = (pinned_array(np.uint8, 2 * key_bytes + 4096), pinned_array(np.uint32, 2 * rows + 1024),
                      pinned_array(np.uint64, 2 * rows + 1024))
        try:
            blob, lens, counts = table.export(out=result)
        except capi.WfcuError:
            blob, lens, counts = table.export()
        d2h = blob.nbytes + lens.nbytes + counts.nbytes
    e2e_step()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    barrier()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    t = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = job_bytes / float(t.item()) / 1e9
    # context for the end-to-end number: a bare pinned host -> device copy of the same shard
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record()
    dev.copy_(host, non_blocking=True)
    c1.record()
    torch.cuda.synchronize()
    h2d_gbps = nbytes / (c0.elapsed_time(c1) * 1e-3) / 1e9 if nbytes else 0.0

    if rank == 0:
        peak, peak_src = measured_peak_gbs()
        k_ms = kernel_ms / max(kernel_launches, 1)
        achieved = nbytes / (k_ms * 1e-3) / 1e9 if k_ms > 0 else 0.0
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": w["scaling"], "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": w["name"], "vocab": w["vocab"], "zipf_s": ZIPF_S, "doc_bytes": DOC_BYTES,
                       "seed": SEED, "documents": total_docs, "bytes_per_gpu": nbytes, "job_bytes": job_bytes,
                       "tokens": job_tokens, "distinct_words": job_distinct,
                       "parallelism": f"document shard d mod {world}" + (", hash-partitioned all-to-all merge" + (" (no host sync per step" + (", exchange of step k on a second stream under the count of step k+1" if overlap and ax is not None else "") + ")" if ax is not None else "") if world > 1 else ""),
                       "l2": f"inputs ({nbytes / 1e9:.2f} GB per GPU) larger than the 126 MB L2; no flush needed" if nbytes > (252 << 20) else f"inputs of {nbytes / 1e6:.0f} MB per GPU: NOT larger than twice the 126 MB L2 (reduced --docs run)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "traffic": ncu_traffic("wc_count_kernel", nbytes, w["vocab"]),
                         "traffic_source": ("static: ncu --set full capture of this kernel on this config (profiles/traffic.json), not re-measured in this run"
                                            if ncu_traffic("wc_count_kernel", nbytes, w["vocab"]) is not None else
                                            "none: no committed ncu capture for this shard size / vocabulary"),
                         "kernel": "wc_count_kernel", "kernel_ms": k_ms, "kernel_launches": kernel_launches,
                         "algorithmic_bytes_per_launch": nbytes, "peak_source": peak_src},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps, "api": "wfcu_counter_count_host + wfcu_counter_export",
                    "bare_pinned_h2d_copy_GBps_per_gpu": h2d_gbps},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        line["host_numa"] = numa
        if world == 1 and not args.no_cpu:
            os.sched_setaffinity(0, all_cpus)      # the CPU baseline gets every core of the box
            line["cpu_baseline"], k_docs, ref_table = cpu_baseline(capi, w["vocab"], total_docs)
            line["parity"] = parity_check(capi, dev.data_ptr(), min(k_docs, len(my_docs)), slots, ref_table)
            if not line["parity"]["equal"]:
                print("PARITY FAILURE: the device table differs from the reference's", file=sys.stderr)
        if not args.no_mapreduce:
            line["extra"] = {"mapreduce": mapreduce_line(capi, torch, device, stream, peak, world == 1 and not args.no_cpu),
                             "sanitize": sanitize_line(capi, torch, dev, nbytes, peak),
                             "non_ascii": non_ascii_line(capi, torch, device, stream, peak)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_cfg5(args) -> None:
    """BASELINE.json config 5 on one GPU: four synthetic speakers -> per-speaker top-k and distinctive words."""
    import numpy as np
    import torch
    from paper_2206_05269_b200 import capi
    import oracle
    if max(args.gpus, 1) != 1 or int(os.environ.get("WORLD_SIZE", "1")) != 1:
        raise SystemExit("bench.py: --workload cfg5 runs on one GPU (the four tables and their pooled complements are rank-local)")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: the product has no CPU path")
    torch.cuda.set_device(0)
    device = torch.device("cuda", 0)
    speakers, vocab, k = [1, 2, 3, 4], 1000000, 25
    docs = args.docs or 954
    stream = torch.cuda.current_stream(device).cuda_stream
    dev = {}
    for sp in speakers:
        host = torch.empty(docs * DOC_BYTES, dtype=torch.uint8).pin_memory()
        capi.synth_corpus_strided(SEED, 0, 1, docs, vocab, ZIPF_S, sp, DOC_BYTES, out=host.numpy())
        dev[sp] = host.to(device)
    torch.cuda.synchronize()
    counters = {sp: capi.Counter(table_slots=1 << 22) for sp in speakers}
    pooled = {sp: capi.Counter(table_slots=1 << 23) for sp in speakers}
    nbytes = docs * DOC_BYTES * len(speakers)
    report = {}

    def step():
        for sp in speakers:
            counters[sp].reset(stream)
            counters[sp].count_dev(dev[sp].data_ptr(), docs * DOC_BYTES, stream)
        for sp in speakers:
            pooled[sp].reset(stream)
            for o in speakers:
                if o != sp:
                    pooled[sp].merge(counters[o], stream)
            report[sp] = (counters[sp].top_k(k, stream), counters[sp].distinctive(pooled[sp], k, stream))

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launches0 = capi.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clocks:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    launches = capi.launch_count() - launches0
    # parity on a bounded sample: the first documents of every speaker, reports against the oracle
    sample_docs = 4
    small, cpu = {}, {}
    for sp in speakers:
        small[sp] = capi.Counter(table_slots=1 << 20)
        small[sp].count_dev(dev[sp].data_ptr(), sample_docs * DOC_BYTES)
        cpu[sp] = oracle.port().wordcount([dev[sp][:sample_docs * DOC_BYTES].cpu().numpy()])
    equal = True
    for sp in speakers:
        others_dev = capi.Counter(table_slots=1 << 21)
        others_cpu = {}
        for o in speakers:
            if o != sp:
                others_dev.merge(small[o])
                for wd, c in cpu[o].items():
                    others_cpu[wd] = others_cpu.get(wd, 0) + c
        equal &= small[sp].top_k(k) == oracle.port().top_k(cpu[sp], k)
        equal &= small[sp].distinctive(others_dev, k) == oracle.port().distinctive(cpu[sp], others_cpu, k)
    line = {
        "metric": METRIC, "value": nbytes / (ms * 1e-3) / 1e9, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": {"workload": "four synthetic speaker corpora (1 M-word vocabulary, 1 % speaker-specific words), counted, pooled and "
                               "reported (top-25, 25 most distinctive words per speaker) on 1 GPU",
                   "speakers": len(speakers), "documents_per_speaker": docs, "job_bytes": nbytes, "k": k,
                   "distinct_words_per_speaker": [counters[sp].stats()[0] for sp in speakers],
                   "most_distinctive": {str(sp): report[sp][1][0][0].decode("utf-8", "replace") for sp in speakers},
                   "l2": "inputs (4 x 1 GB) larger than the 126 MB L2; no flush needed"},
        "parity": {"checked": True, "docs_per_speaker": sample_docs, "equal": bool(equal),
                   "against": "oracle top_k / distinctive_words (words, counts and doubles) on the same bytes"},
        "gpu_launches": int(launches), "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def mapreduce_line(capi, torch, device, stream, peak, with_cpu: bool) -> dict:
    """BASELINE.json config 2: sum of f(x) over 2^28 fp32 (1 GiB), f = identity and x^2.
    Input = the reference bench's recipe (proj/src/cli.cpp:122-124: mt19937_64(seed 1), uniform(0,1)), rounded to
    fp32.  Per map: resident + CUDA-event timed (GBps), checked against the oracle's serial fold
    (engine.cpp:82-86 on the widened values; 1e-5 relative is the bar), end to end through wfcu_map_reduce_host from
    pinned host memory (e2e_GBps, H2D inside), and the reference's own map_reduce_serial / map_reduce_blocked{256,
    all cores} on this box's host cores (MapKind has no x^2: the CPU figures are the identity map's)."""
    import numpy as np
    import oracle
    n = 1 << 28
    host = torch.empty(n, dtype=torch.float32).pin_memory()
    xh = host.numpy()
    xh[:] = capi.synth_uniform(SEED, n, np.float32)
    x = host.to(device, non_blocking=True)
    out = torch.zeros(1, device=device, dtype=torch.float64)
    res = {}
    for name, kind in (("identity", capi.MAP_IDENTITY), ("square", capi.MAP_SQUARE)):
        for _ in range(3):
            capi.map_reduce_dev_async(x.data_ptr(), capi.DTYPE_F32, n, kind, out.data_ptr(), 0, stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            capi.map_reduce_dev_async(x.data_ptr(), capi.DTYPE_F32, n, kind, out.data_ptr(), 0, stream)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        got = float(out.item())
        ref = oracle.port().map_reduce_serial(xh, kind)
        capi.map_reduce_host(xh, kind)
        t0 = time.perf_counter()
        e2e_got = 0.0
        for _ in range(3):
            e2e_got = capi.map_reduce_host(xh, kind)
        e2e_s = (time.perf_counter() - t0) / 3
        res[name] = {"ms": ms, "GBps": 4 * n / ms / 1e6, "frac_of_hbm_peak": 4 * n / ms / 1e6 / peak,
                     "value": got, "oracle_serial_fold": ref, "rel_err_vs_oracle": abs(got - ref) / max(1.0, abs(ref)),
                     "e2e_GBps": 4 * n / e2e_s / 1e9, "e2e_rel_err_vs_oracle": abs(e2e_got - ref) / max(1.0, abs(ref)),
                     "e2e_api": "wfcu_map_reduce_host (pinned host fp32 -> H2D -> reduce -> scalar)"}
    line = {"config": "sum f(x) over 2^28 fp32, mt19937_64(1) uniform(0,1) (reference bench recipe), 1 GiB, 1 GPU", **res}
    if with_cpu and oracle.ref_available():
        cores = os.cpu_count() or 1
        m = 1 << 26      # bounded sample: 2^26 doubles (the reference's spans are fp64)
        xd = xh[:m].astype(np.float64)
        t0 = time.perf_counter()
        v1 = oracle.ref().map_reduce_serial(xd, capi.MAP_IDENTITY)
        t1 = time.perf_counter()
        v2 = oracle.ref().map_reduce_blocked(xd, capi.MAP_IDENTITY, 256, cores)
        t2 = time.perf_counter()
        line["cpu_baseline"] = {"kind": "reference", "sample": f"first 2^26 of the 2^28 values, widened to fp64 ({8 * m >> 20} MiB)",
                                "map_reduce_serial": {"GBps_of_fp64": 8 * m / (t1 - t0) / 1e9, "cores": 1, "value": v1},
                                "map_reduce_blocked_256": {"GBps_of_fp64": 8 * m / (t2 - t1) / 1e9, "cores": cores, "value": v2}}
    return line


def non_ascii_line(capi, torch, device, stream, peak) -> dict:
    """Text that is not ASCII: the first 256 documents of the cfg3 corpus with bigrams replaced by
    two-byte letters (accented), by U+2019 inside words (typographic), by three-byte letters in 13 % / 97 % of the
    words (kana).  Resident, CUDA-event timed; all of them are counted exactly (tests/test_gpu_count_kernel.py)."""
    import numpy as np
    base = capi.synth_corpus(SEED, 0, 256, 50000, ZIPF_S, 0, DOC_BYTES).tobytes()
    kana = list(zip((b"ba", b"ca", b"da", b"fa", b"ga", b"a", b"e", b"i"), "あいうえお漢字語"))
    flavours = {
        "accented": [(b"ba", "é"), (b"ca", "ü"), (b"da", "ö"), (b"fa", "ß"), (b"ga", "ñ")],
        "typographic": [(a, a[:1].decode() + "’" + a[1:].decode()) for a in (b"ab", b"ba", b"ca")],
        "kana_13pct": kana[:5],
        "kana_97pct": kana,
    }
    res = {}
    for name, subs in flavours.items():
        raw = base
        for a, b in subs:
            raw = raw.replace(a, b.encode())
        raw = raw[:len(raw) & ~15]
        dev = torch.from_numpy(np.frombuffer(raw, dtype=np.uint8).copy()).to(device)
        c = capi.Counter(table_slots=1 << 21, deferred_slots=1 << 27)
        for _ in range(3):
            c.reset(stream); c.count_dev(dev.data_ptr(), dev.numel(), stream)
        torch.cuda.synchronize()
        c.status()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            c.reset(stream); c.count_dev(dev.data_ptr(), dev.numel(), stream)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        distinct, tokens, _ = c.stats()
        res[name] = {"bytes": dev.numel(), "ms": ms, "GBps": dev.numel() / ms / 1e6, "frac_of_hbm_peak": dev.numel() / ms / 1e6 / peak,
                     "tokens": tokens, "distinct_words": distinct}
        c.close()
    return {"config": "first 256 cfg3 documents with bigrams replaced by non-ASCII letters, 1 GPU, resident", **res}


def sanitize_line(capi, torch, dev, nbytes, peak) -> dict:
    """The ingest step in front of the path (utf8_sanitize) on the resident shard:
    the valid corpus as it is, and with 0xFF planted every 1000 bytes.  Algorithmic bytes = input read
    once + output written once; the call includes its one host read (the output length)."""
    out = torch.empty(nbytes + nbytes // 400 + 64, dtype=torch.uint8, device=dev.device)
    res = {}
    for name in ("valid", "1_in_1000_invalid"):
        src = dev
        if name != "valid":
            src = dev.clone()
            src[500::1000] = 0xFF
        m = 0
        for _ in range(3):
            m = capi.utf8_sanitize_dev(src.data_ptr(), nbytes, out.data_ptr(), out.numel())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            capi.utf8_sanitize_dev(src.data_ptr(), nbytes, out.data_ptr(), out.numel())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[name] = {"ms": ms, "input_GBps": nbytes / ms / 1e6, "algorithmic_GBps": (nbytes + m) / ms / 1e6,
                     "frac_of_hbm_peak": (nbytes + m) / ms / 1e6 / peak, "out_bytes": m}
    return {"config": "utf8_sanitize of the resident 1 GB shard, 1 GPU", **res}


def self_launch_cmd(gpus: int, argv: list[str], port: int | None = None) -> list[str]:
    """`python bench.py --gpus N` outside torchrun: the command that runs it as one rank per GPU."""
    if port is None:
        import socket
        with socket.socket() as sock:
            sock.bind(("127.0.0.1", 0))
            port = sock.getsockname()[1]
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *argv]


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + ["cfg5"], default="cfg3")
    ap.add_argument("--docs", type=int, default=None, help="override document count (per GPU for cfg3, total for cfg4)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-overlap-exchange", action="store_true",
                    help="N > 1: keep the all-to-all and the merge on the counting stream (default: a second stream, "
                         "overlapping the next step's count)")
    ap.add_argument("--sync-exchange", action="store_true",
                    help="N > 1: use the merge that reads the region sizes on the host every step")
    ap.add_argument("--sample-docs", type=int, default=None, help="reference arm: documents per step")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="collective backend at N > 1 (gloo only for single-GPU testing of the N > 1 path)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-mapreduce", action="store_true", help="skip the config-2 map-reduce extra")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        # one rank per GPU: re-run under torch.distributed.run (NCCL's init lines stay on: they name every rank)
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        raise SystemExit(subprocess.call(self_launch_cmd(args.gpus, sys.argv[1:]), env=env))
    # the native libraries are built in-tree; make sure they exist and are current (rank 0 builds, a no-op when fresh)
    from paper_2206_05269_b200 import build as native
    if int(os.environ.get("LOCAL_RANK", "0")) == 0:
        native.build_all()
    else:
        for _ in range(600):
            if (native.LIB / "libwfcu.so").exists():
                break
            time.sleep(0.5)
    if args.workload == "cfg5":
        if args.impl == "reference":
            raise SystemExit("bench.py: the reference arm times cfg3 / cfg4 (run_wordcount); cfg5's reports are checked inside the b200 arm")
        run_cfg5(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()

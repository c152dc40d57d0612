"""CPU: bench.py's reference arm runs here (no GPU) and prints the contract's JSON line."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--sample-docs", "2"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "wordcount_corpus_GBps" and d["unit"] == "GB/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["vs_baseline"] is None
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("word count")


def test_reference_arm_other_ranks_do_nothing():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2"],
                         capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_reference_arm_does_not_map_the_cuda_library():
    """The reference process builds its corpus with oracle/libwfsynth.so: libwfcu.so never enters its address space."""
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0','--sample-docs','1'];"
            "runpy.run_path(r'%s', run_name='__main__')" % os.path.join(ROOT, "bench.py"))
    probe = code + "\nmaps=open('/proc/self/maps').read()\nprint('MAPPED_WFCU' if 'libwfcu.so' in maps else 'CLEAN', file=sys.stderr)"
    out = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "CLEAN" in out.stderr and "MAPPED_WFCU" not in out.stderr
    d = json.loads([l for l in out.stdout.splitlines() if l.strip()][0])
    assert d["config"]["same_config"] is False      # --sample-docs 1 of 954


def test_gpus_n_self_launches_one_rank_per_gpu():
    """`python bench.py --gpus N` outside torchrun re-runs itself under torch.distributed.run with N ranks."""
    sys.path.insert(0, ROOT)
    import bench
    cmd = bench.self_launch_cmd(4, ["--gpus", "4", "--steps", "2"], port=29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"] and cmd[-5].endswith("bench.py")
    # and the launch really happens: without GPUs every rank stops at "needs a CUDA device", after the rendezvous
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--no-cpu"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode != 0
    assert out.stderr.count("bench.py needs a CUDA device") >= 2 or "torch.distributed" in out.stderr

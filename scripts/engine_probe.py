"""Developer probe: the reference-named engine calls (bit-exact serial / blocked fold) at cfg2 size on the device,
next to the roofline reduction and the reference's CPU code."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2206_05269_b200 import capi

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
x = capi.synth_uniform(1, n, np.float64)
dx = torch.from_numpy(x).cuda()
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): v = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps, v
for kind, name in ((capi.MAP_IDENTITY, "identity"), (capi.MAP_SQUARE_ROOT, "sqrt")):
    t_fast, v_fast = timed(lambda: capi.map_reduce_dev(dx.data_ptr(), capi.DTYPE_F64, n, kind))
    t_blk, v_blk = timed(lambda: capi.map_reduce_blocked_dev(dx.data_ptr(), capi.DTYPE_F64, n, kind, 256))
    t_ser, v_ser = timed(lambda: capi.map_reduce_blocked_dev(dx.data_ptr(), capi.DTYPE_F64, n, kind, n), reps=1)
    line = f"{name}: n=2^{n.bit_length()-1} fp64 | fast {t_fast*1e3:.3f} ms ({8*n/t_fast/1e9:.0f} GB/s) | blocked{{256}} {t_blk*1e3:.3f} ms ({8*n/t_blk/1e9:.0f} GB/s) | serial (one block) {t_ser*1e3:.1f} ms ({8*n/t_ser/1e9:.2f} GB/s)"
    if oracle.ref_available() and n <= 1 << 28:
        r = oracle.ref()
        t0 = time.perf_counter(); c_ser = r.map_reduce_serial(x, kind); t1 = time.perf_counter()
        c_blk = r.map_reduce_blocked(x, kind, 256, os.cpu_count()); t2 = time.perf_counter()
        line += f" | CPU reference serial {1e3*(t1-t0):.0f} ms, blocked{{256,{os.cpu_count()}}} {1e3*(t2-t1):.0f} ms | bit-equal: serial {v_ser == c_ser}, blocked {v_blk == c_blk}, fast rel err {abs(v_fast-c_ser)/abs(c_ser):.1e}"
    print(line, flush=True)

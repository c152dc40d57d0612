"""GPU parity: map-then-reduce engine vs the oracle (reference: proj/src/engine.cpp)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5   # BASELINE.json north_star: 1e-5 relative against the reference's sum


def rel(a, b):
    return abs(a - b) / max(1.0, abs(b))


def test_reference_goldens(capi, cuda):
    v = np.array([1.0, 4.0, 9.0])
    assert capi.map_reduce_host(v, capi.MAP_SQUARE_ROOT) == 6.0                       # engine_test.cpp:24-29
    assert capi.map_reduce_host(np.zeros(0), capi.MAP_SQUARE_ROOT) == 0.0
    assert capi.map_reduce_host(np.zeros(0), capi.MAP_IDENTITY) == 0.0
    assert capi.map_reduce_blocked_host(v, capi.MAP_SQUARE_ROOT, 1) == 6.0            # :31-36
    assert capi.map_reduce_blocked_host(np.zeros(0), capi.MAP_IDENTITY, 16) == 0.0
    assert capi.alternating_harmonic(0) == 0.0 and capi.alternating_harmonic(1) == 1.0    # :57-61
    assert capi.alternating_harmonic(2) == 0.5
    ten = capi.map_reduce_blocked_host(np.zeros(10), capi.MAP_ALTERNATING_HARMONIC_TERM, 10)
    assert abs(ten - 0.6456349206349207) <= 1e-15                                      # :47-55
    assert abs(capi.alternating_harmonic(10 ** 6) - 0.6931471805599453) <= 1e-6        # acceptance_test.cpp:259-261
    assert np.isnan(capi.map_reduce_host(np.array([4.0, -1.0]), capi.MAP_SQUARE_ROOT))  # :104-108
    with pytest.raises(capi.InvalidArgument):                                           # :110-116
        capi.map_reduce_blocked_host(np.ones(1), capi.MAP_IDENTITY, 0)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [0, 1, 2, 3, 5, 1023, 1024, 1025, 100000, (1 << 20) + 3])
def test_fast_reduce_matches_serial(capi, cuda, port, dtype, n):
    x = capi.synth_uniform(1, n, dtype)
    for kind in (capi.MAP_IDENTITY, capi.MAP_SQUARE_ROOT, capi.MAP_ALTERNATING_HARMONIC_TERM, capi.MAP_SQUARE):
        got = capi.map_reduce_host(x, kind)
        want = port.map_reduce_serial(x, kind)
        assert rel(got, want) <= REL_TOL, (kind, got, want)
        assert rel(got, want) <= 1e-12    # what fp64 accumulation actually delivers
        assert capi.map_reduce_host(x, kind) == got   # run-to-run bitwise reproducible


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_blocked_engine_is_bit_exact(capi, cuda, port, dtype):
    """wfcu_map_reduce_blocked_* == reference map_reduce_blocked, bit for bit (engine_test.cpp:81-93)"""
    x = capi.synth_uniform(555, 100000, dtype)
    for kind in (capi.MAP_IDENTITY, capi.MAP_SQUARE_ROOT, capi.MAP_ALTERNATING_HARMONIC_TERM, capi.MAP_SQUARE):
        for block in (1, 7, 256, 100000, 100100):
            assert capi.map_reduce_blocked_host(x, kind, block) == port.map_reduce_blocked(x, kind, block), (kind, block)
    # one covering block == serial fold, bitwise (engine_test.cpp:38-45)
    y = capi.synth_uniform(9001, 1537, dtype)
    for kind in (capi.MAP_IDENTITY, capi.MAP_SQUARE_ROOT):
        assert capi.map_reduce_blocked_host(y, kind, y.size) == port.map_reduce_serial(y, kind)


def test_position_base_splits_the_series(capi, cuda, port):
    """a rank holding a slice passes its offset: partial sums add up to the whole"""
    n = 100003
    whole = capi.map_reduce_dev(0, capi.DTYPE_F64, n, capi.MAP_ALTERNATING_HARMONIC_TERM)
    parts = sum(capi.map_reduce_dev(0, capi.DTYPE_F64, hi - lo, capi.MAP_ALTERNATING_HARMONIC_TERM, position_base=lo)
                for lo, hi in ((0, 30000), (30000, 77777), (77777, n)))
    assert rel(parts, whole) <= 1e-13
    assert rel(whole, port.alternating_harmonic(n)) <= 1e-12


def test_headline_config_square_sum(capi, cuda, port):
    """BASELINE.json config 2 shape (scaled to 2^24 for the CPU check): sum x^2 over fp32"""
    x = capi.synth_uniform(1, 1 << 24, np.float32)
    dx = cuda.from_numpy(x).cuda()
    got = capi.map_reduce_dev(dx.data_ptr(), capi.DTYPE_F32, dx.numel(), capi.MAP_SQUARE)
    assert rel(got, port.map_reduce_serial(x, capi.MAP_SQUARE)) <= REL_TOL


def test_headline_config_full_size(capi, cuda, port):
    """BASELINE.json config 2 at its full size: sum of x and of x^2 over 2^28 fp32 (the reference bench's
    mt19937_64 / uniform(0,1) recipe, proj/src/cli.cpp:122-124) against the oracle's serial fold
    (proj/src/engine.cpp:15-20, 82-86) within the north star's 1e-5 relative tolerance, and the sum of two
    halves equal to the whole (the split the multi-GPU reduction makes)."""
    n = 1 << 28
    x = capi.synth_uniform(1, n, np.float32)
    dx = cuda.from_numpy(x).cuda()
    for kind in (capi.MAP_IDENTITY, capi.MAP_SQUARE):
        got = capi.map_reduce_dev(dx.data_ptr(), capi.DTYPE_F32, n, kind)
        want = port.map_reduce_serial(x, kind)
        assert rel(got, want) <= 1e-5, (kind, got, want)
        assert rel(got, want) <= 1e-9           # fp64 accumulation; the serial left fold itself drifts by ~sqrt(n) ulp
        half = n // 2
        parts = (capi.map_reduce_dev(dx.data_ptr(), capi.DTYPE_F32, half, kind) +
                 capi.map_reduce_dev(dx.data_ptr() + 4 * half, capi.DTYPE_F32, half, kind, position_base=half))
        assert rel(parts, got) <= 1e-13

"""CPU: the drop-in library links, exports the reference's wfc:: symbols, and refuses to
run without a GPU instead of falling back."""
import subprocess

import pytest


def test_dropin_exports_reference_api(capi):
    so = capi.LIB_PATH.parent / "libwfc_b200.so"
    assert so.exists()
    syms = subprocess.run(["nm", "-D", "--defined-only", "-C", str(so)], capture_output=True, text=True).stdout
    import re
    for name in ("tokenize", "normalize_word", "sort_words", "reduce_sorted", "boundary_repair", "merge_counts",
                 "count_unreduced_words", "run_wordcount", "serial_wordcount", "map_reduce_serial", "map_reduce_blocked",
                 "alternating_harmonic", "top_k", "distinctive_words",
                 # the paper's own exchange and the code-point accessors (wfc/{wire,shuffle,transport,unicode}.hpp)
                 "encode_message", "decode_message", "plan_partition", "encode_outgoing", "exchange_encoded", "exchange",
                 "utf8_decode", "utf8_append", "utf8_sanitize", "utf8_valid", "is_unicode_space", "is_word_char", "simple_lower"):
        assert re.search(r"\bwfc::%s(\[abi:cxx11\])?\(" % name, syms), name


def test_dropin_fails_loudly_without_a_gpu(capi):
    if capi.device_count() > 0:
        pytest.skip("a GPU is visible here")
    exe = capi.LIB_PATH.parent / "wfc_dropin_tests"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert out.returncode != 0
    assert "no CUDA device" in out.stdout + out.stderr

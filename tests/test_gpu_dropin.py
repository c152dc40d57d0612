"""GPU: the C++ drop-in (libwfc_b200.so, the reference's wfc:: API over the C ABI) passes
its reference-style test binary (paper_2206_05269_b200/host/tests/dropin_tests.cpp)."""
import subprocess

import pytest

pytestmark = pytest.mark.gpu


def test_dropin_binary(capi, cuda):
    exe = capi.LIB_PATH.parent / "wfc_dropin_tests"
    assert exe.exists(), "build the host drop-in first (python -m paper_2206_05269_b200.build)"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-1000:]
    assert "0 failed" in out.stdout


REF_SUITES = ["text", "reduce", "engine", "pipeline", "analysis", "shuffle", "wire"]


@pytest.mark.parametrize("suite", REF_SUITES)
def test_reference_suite_unmodified(capi, cuda, suite):
    """/root/reference/proj/tests/<suite>_test.cpp, compiled UNMODIFIED from where it lies against the drop-in
    (paper_2206_05269_b200/build.py::build_reference_suites; doctest macros from tests/shim/doctest.h), passes on
    the GPU: every TEST_CASE of the reference's own suite, with its own goldens."""
    exe = capi.LIB_PATH.parent / "reftests" / f"{suite}_test"
    assert exe.exists(), "lib/reftests is built where /root/reference is present and travels with the snapshot"
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    assert "| 0 failed" in out.stdout


def test_relink_with_the_references_own_report_cpp(capi, cuda, tmp_path):
    """INTEGRATION.md section 1 tried for real: the reference's report.cpp (unmodified) + a caller written against
    the reference's headers, linked with libwfc_b200.so, prints the byte-exact golden table of
    proj/tests/cli_test.cpp:51-60 for the two-document fixture, and the JSON form through the reference's
    frequency_json."""
    import json
    import os
    exe = capi.LIB_PATH.parent / "reftests" / "relink_demo"
    if not exe.exists():
        pytest.skip("relink demo not built (no json.hpp in this image)")
    fixtures = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fixtures.json")))
    two = tmp_path / "two-docs"
    two.mkdir()
    for i, hexdoc in enumerate(fixtures["two-docs"]["docs"]):
        (two / f"doc{i + 1}.txt").write_bytes(bytes.fromhex(hexdoc))
    (two / "ignored.md").write_text("not a text file")
    out = subprocess.run([str(exe), "wordcount", str(two), "2", "tsv"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout == ("mapreduce\t2\t0.166666666667\ntest\t2\t0.166666666667\nto\t2\t0.166666666667\n"
                          "a\t1\t0.0833333333333\nalgorithm\t1\t0.0833333333333\ncool\t1\t0.0833333333333\n"
                          "i\t1\t0.0833333333333\nis\t1\t0.0833333333333\nwant\t1\t0.0833333333333\n")
    assert [l.split("\t")[:2] for l in out.stderr.splitlines()][-1] == ["timing", "total"]
    js = subprocess.run([str(exe), "wordcount", str(two), "3", "json"], capture_output=True, text=True, timeout=300)
    assert js.returncode == 0, js.stderr
    rows = json.loads(js.stdout)      # frequency_json (proj/src/report.cpp:19-25): an array of {word, count, relfreq}
    assert len(rows) == 9 and rows[0] == {"word": "mapreduce", "count": 2, "relfreq": 2 / 12}
    bad = subprocess.run([str(exe), "wordcount", str(tmp_path / "missing"), "2"], capture_output=True, text=True, timeout=300)
    assert bad.returncode == 1 and "not a readable directory" in bad.stderr


def test_one_caller_two_libraries(capi, cuda):
    """tests/relink/api_bench.cpp includes only wfc/ headers and is linked twice: with libwfc_b200.so and (in the build
    container, travelling as oracle/_ref/api_bench_ref) with the unmodified reference.  Every result of the public API
    -- the merged counts, the serial count, the pre-repair shards of run_wordcount(corpus, n), the tokens of a document
    in text order, top-25, the bit-exact blocked fold -- must be identical between the two processes."""
    import json
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ours = capi.LIB_PATH.parent / "reftests" / "api_bench_b200"
    ref = os.path.join(root, "oracle", "_ref", "api_bench_ref")
    assert ours.exists() and os.path.exists(ref), "built where /root/reference is present; travels with the snapshot"
    for docs, workers in ((3, 1), (8, 3)):
        a = subprocess.run([str(ours), str(docs), str(workers), "1"], capture_output=True, text=True, timeout=600)
        b = subprocess.run([ref, str(docs), str(workers), "1"], capture_output=True, text=True, timeout=600)
        assert a.returncode == 0 and b.returncode == 0, a.stderr[-2000:] + b.stderr[-2000:]
        ja, jb = json.loads(a.stdout), json.loads(b.stdout)
        for key in ("counts", "counts_checksum", "serial_checksum", "pre_repair_checksum", "tokens_doc0", "tokens_checksum",
                    "top25_checksum", "fold"):
            assert ja[key] == jb[key], (key, ja[key], jb[key])

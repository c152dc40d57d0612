"""In-tree build of the native libraries (nvcc for sm_100a, g++ for the host shim).

  paper_2206_05269_b200/lib/libwfcu.so      CUDA kernels + the C ABI of include/wfcu.h
  paper_2206_05269_b200/lib/libwfc_b200.so  C++ drop-in for the reference's wfc:: API
                                            (host/include/wfc/*.hpp) on top of the C ABI
  paper_2206_05269_b200/lib/wfc_dropin_tests  the reference-style C++ test binary

The outputs are git-ignored but travel to the GPU box with the gpurun snapshot.
`python -m paper_2206_05269_b200.build` rebuilds when a source is newer than the output.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
HOST = PKG / "host"
LIB = PKG / "lib"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-fvisibility=hidden,-O2",
    "--expt-relaxed-constexpr",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA extension cannot be built")


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _run(cmd: list[str]) -> None:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + proc.stdout + proc.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} (exit {proc.returncode})")


def build_wfcu(force: bool = False, verbose: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libwfcu.so"
    cu = sorted(CSRC.glob("*.cu"))
    cpp = sorted(CSRC.glob("*.cpp"))
    hdr = sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "wfcu.h"]
    if not force and not _stale(out, cu + cpp + hdr):
        return out
    objs = []
    obj_dir = LIB / "obj"
    obj_dir.mkdir(exist_ok=True)
    for src in cu + cpp:
        obj = obj_dir / (src.name + ".o")
        if force or _stale(obj, [src] + hdr):
            cmd = [_nvcc(), *NVCC_FLAGS, *os.environ.get("WFCU_NVCC_EXTRA", "").split(), "-c", str(src), "-o", str(obj)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            _run(cmd)
        objs.append(str(obj))
    _run([_nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(out), *objs,
          "-Xlinker", "--no-undefined", "-lpthread"])
    return out


def build_host(force: bool = False) -> Path | None:
    """C++ drop-in (libwfc_b200.so) and its test binary; needs libwfcu.so first."""
    if not HOST.exists():
        return None
    LIB.mkdir(exist_ok=True)
    out = LIB / "libwfc_b200.so"
    srcs = sorted((HOST / "src").glob("*.cpp"))
    hdrs = sorted((HOST / "include" / "wfc").glob("*.hpp")) + [ROOT / "include" / "wfcu.h"]
    cxx = os.environ.get("CXX") or shutil.which("g++") or "g++"
    common = [cxx, "-std=c++20", "-O2", "-fPIC", "-pthread", "-ffp-contract=off", f"-I{HOST / 'include'}", f"-I{ROOT / 'include'}"]
    if force or _stale(out, srcs + hdrs + [LIB / "libwfcu.so"]):
        _run(common + ["-shared", "-o", str(out), *map(str, srcs), f"-L{LIB}", "-lwfcu", "-Wl,-rpath,$ORIGIN"])
    tests = sorted((HOST / "tests").glob("*.cpp"))
    if tests:
        exe = LIB / "wfc_dropin_tests"
        if force or _stale(exe, tests + hdrs + [out]):
            _run(common + ["-o", str(exe), *map(str, tests), f"-L{LIB}", "-lwfc_b200", "-lwfcu", "-Wl,-rpath,$ORIGIN"])
    return out


REF_TESTS = Path("/root/reference/proj/tests")
REF_SUITES = ["text", "reduce", "engine", "pipeline", "analysis", "shuffle", "wire"]


def build_reference_suites(force: bool = False) -> list[Path]:
    """The reference's OWN test files (proj/tests/*_test.cpp + support.hpp), compiled unmodified from where they
    lie against libwfc_b200.so: the drop-in headers stand in for proj/include, tests/shim/doctest.h for the
    vendored doctest the reference tree does not ship.  Binaries land in lib/reftests/ and travel to the GPU
    box; nothing of the reference is copied.  No-op where /root/reference is absent (the GPU box)."""
    out_dir = LIB / "reftests"
    if not REF_TESTS.exists() or not (LIB / "libwfc_b200.so").exists():
        return sorted(out_dir.glob("*_test")) if out_dir.exists() else []
    out_dir.mkdir(exist_ok=True)
    cxx = os.environ.get("CXX") or shutil.which("g++") or "g++"
    shim = ROOT / "tests" / "shim"
    deps = sorted((HOST / "include" / "wfc").glob("*.hpp")) + [shim / "doctest.h", LIB / "libwfc_b200.so"]
    built = []
    for name in REF_SUITES:
        src = REF_TESTS / f"{name}_test.cpp"
        exe = out_dir / f"{name}_test"
        if force or _stale(exe, [src, REF_TESTS / "support.hpp"] + deps):
            _run([cxx, "-std=c++20", "-O1", "-pthread", f"-I{shim}", f"-I{HOST / 'include'}", f"-I{REF_TESTS}",
                  '-DWFC_FIXTURES_DIR="/root/reference/proj/fixtures"', "-o", str(exe), str(src),
                  f"-L{LIB}", "-lwfc_b200", "-lwfcu", "-Wl,-rpath,$ORIGIN/.."])
        built.append(exe)
    return built


def build_relink_demo(force: bool = False) -> Path | None:
    """INTEGRATION.md section 1, tried for real: the reference's own report.cpp (unmodified, compiled where it lies,
    against ITS wfc/report.hpp -- reached through a symlink so that every other wfc/ header comes from the drop-in) +
    tests/relink/relink_main.cpp (the cli.cpp flows without CLI11) + libwfc_b200.so.  nlohmann's json.hpp is the
    copy the image carries (cudnn_frontend's thirdparty directory); without it the demo is skipped."""
    ref = Path("/root/reference/proj")
    out_dir = LIB / "reftests"
    exe = out_dir / "relink_demo"
    if not ref.exists() or not (LIB / "libwfc_b200.so").exists():
        return exe if exe.exists() else None
    json_dirs = [Path(p) for p in sys.path if p and (Path(p) / "include/cudnn_frontend/thirdparty/nlohmann/json.hpp").exists()]
    if not json_dirs:
        return None
    json_inc = json_dirs[0] / "include/cudnn_frontend/thirdparty/nlohmann"
    out_dir.mkdir(exist_ok=True)
    view = out_dir / "relink_include" / "wfc"          # the one header a maintainer keeps from proj/include
    view.mkdir(parents=True, exist_ok=True)
    link = view / "report.hpp"
    if not link.exists():
        link.symlink_to(ref / "include/wfc/report.hpp")
    main = ROOT / "tests" / "relink" / "relink_main.cpp"
    deps = [main, ref / "src/report.cpp", LIB / "libwfc_b200.so"] + sorted((HOST / "include" / "wfc").glob("*.hpp"))
    if force or _stale(exe, deps):
        cxx = os.environ.get("CXX") or shutil.which("g++") or "g++"
        _run([cxx, "-std=c++20", "-O1", "-pthread", f"-I{view.parent}", f"-I{HOST / 'include'}", f"-I{json_inc}",
              "-o", str(exe), str(main), str(ref / "src/report.cpp"), f"-L{LIB}", "-lwfc_b200", "-lwfcu",
              "-Wl,-rpath,$ORIGIN/.."])
    return exe


def build_api_bench(force: bool = False) -> Path | None:
    """tests/relink/api_bench.cpp -- a caller of the public wfc:: API that includes only wfc/ headers -- linked with the
    drop-in (its twin oracle/_ref/api_bench_ref, linked with the reference, is built by oracle/Makefile)."""
    out_dir = LIB / "reftests"
    exe = out_dir / "api_bench_b200"
    main = ROOT / "tests" / "relink" / "api_bench.cpp"
    if not (LIB / "libwfc_b200.so").exists() or not main.exists():
        return None
    out_dir.mkdir(exist_ok=True)
    deps = [main, LIB / "libwfc_b200.so"] + sorted((HOST / "include" / "wfc").glob("*.hpp"))
    if force or _stale(exe, deps):
        cxx = os.environ.get("CXX") or shutil.which("g++") or "g++"
        _run([cxx, "-std=c++20", "-O2", "-pthread", f"-I{HOST / 'include'}", "-o", str(exe), str(main),
              f"-L{LIB}", "-lwfc_b200", "-lwfcu", "-Wl,-rpath,$ORIGIN/.."])
    return exe


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_wfcu(force, verbose)
    build_host(force)
    build_reference_suites(force)
    build_relink_demo(force)
    build_api_bench(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print("built:", *(p.name for p in sorted(LIB.glob("*")) if p.is_file()))

"""In-tree native build (no JIT cache): the .so files land under
paper_2605_23057_b200/lib/ and oracle/, so gpurun ships them to the B200 box.

  libmodeswitch.so   host controller (C++20) + executor, C ABI in include/msw_host.h
  libmsw_engine.so   sm_100a CUDA engine, C ABI in include/msw_engine.h
  oracle/liboracle.so, oracle/_ref/*  test-only checkers (built by build_oracle)
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "lib")
INC = os.path.join(ROOT, "include")
CSRC = os.path.join(PKG, "csrc")
# nlohmann/json 3.11.3 (the version the reference's byte-exact NDJSON goldens
# were generated with). MSW_NLOHMANN_INCLUDE names a directory holding
# json.hpp; otherwise the copy vendored by cudnn_frontend in this image.
NLOHMANN_CANDIDATES = [
    os.environ.get("MSW_NLOHMANN_INCLUDE", ""),
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann",
    "/usr/include/nlohmann",
]
NLOHMANN_VERSION = (3, 11, 3)


def nlohmann_dir() -> str:
    import re
    for d in NLOHMANN_CANDIDATES:
        f = os.path.join(d, "json.hpp") if d else ""
        if not f or not os.path.exists(f):
            continue
        txt = open(f, errors="replace").read(200_000)
        ver = tuple(int(re.search(rf"#define NLOHMANN_JSON_VERSION_{k} (\d+)", txt).group(1))
                    for k in ("MAJOR", "MINOR", "PATCH"))
        if ver != NLOHMANN_VERSION:
            raise RuntimeError(f"{f}: nlohmann/json {ver}, need {NLOHMANN_VERSION} "
                               "(byte-exact NDJSON goldens); set MSW_NLOHMANN_INCLUDE")
        return d
    raise RuntimeError("nlohmann/json.hpp 3.11.3 not found; set MSW_NLOHMANN_INCLUDE")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

ENGINE_SO = os.path.join(LIB, "libmsw_engine.so")
HOST_SO = os.path.join(LIB, "libmodeswitch.so")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], cwd: str | None = None) -> None:
    print("[build]", " ".join(cmd[:6]), "...", flush=True)
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} (exit {r.returncode})")


def _headers() -> list[str]:
    return glob.glob(os.path.join(INC, "**", "*.h*"), recursive=True)


def build_engine(force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "engine", "*.cu")))
    deps = srcs + glob.glob(os.path.join(CSRC, "engine", "*.cuh")) + _headers()
    if not srcs:
        raise RuntimeError("no engine sources")
    if force or _stale(ENGINE_SO, deps):
        objdir = os.path.join(ROOT, "build", "engine")
        os.makedirs(objdir, exist_ok=True)
        objs, jobs = [], []
        for s in srcs:
            o = os.path.join(objdir, os.path.basename(s) + ".o")
            objs.append(o)
            if force or _stale(o, [s] + deps[len(srcs):]):
                jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                             "-Xptxas", "-v", "--expt-relaxed-constexpr", "-I", INC,
                             "-I", os.path.join(CSRC, "engine"), "-c", s, "-o", o])
        with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            for f in [ex.submit(_run, j) for j in jobs]:
                f.result()
        _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", ENGINE_SO, *objs,
              "-lpthread", "-ldl", "-lrt"])
    return ENGINE_SO


def build_engine_trace() -> str:
    """Diagnostics build with the MSW_TP timeline probes (-DMSW_TRACE); used
    only by scripts/gemv_timeline.py, never by the product path or tests."""
    out = os.path.join(LIB, "libmsw_engine_trace.so")
    srcs = sorted(glob.glob(os.path.join(CSRC, "engine", "*.cu")))
    objdir = os.path.join(ROOT, "build", "engine_trace")
    os.makedirs(objdir, exist_ok=True)
    objs, jobs = [], []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(o)
        jobs.append([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-DMSW_TRACE", "--expt-relaxed-constexpr", "-I", INC,
                     "-I", os.path.join(CSRC, "engine"), "-c", s, "-o", o])
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        for f in [ex.submit(_run, j) for j in jobs]:
            f.result()
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", out, *objs, "-lpthread", "-ldl", "-lrt"])
    return out


def build_host(force: bool = False) -> str:
    os.makedirs(LIB, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    deps = srcs + _headers() + [ENGINE_SO]
    if force or _stale(HOST_SO, deps):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra",
              "-I", INC, "-I", nlohmann_dir(), *srcs, "-o", HOST_SO,
              "-L", LIB, "-lmsw_engine", "-Wl,-rpath,$ORIGIN", "-lpthread", "-ldl"])
    return HOST_SO


def build_oracle(force: bool = False) -> None:
    odir = os.path.join(ROOT, "oracle")
    _run(["make", "-C", odir, "-j8", "all"] + (["-B"] if force else []))
    if os.path.isdir("/root/reference/proj/core/src"):
        _run(["make", "-C", odir, "-j8", "ref"])


def build_all(force: bool = False) -> None:
    build_engine(force)
    build_host(force)
    build_oracle(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)

"""Build libcommsched.so in-tree: host C++ (g++) + sm_100a kernels (nvcc).

    python -m paper_1803_03288_b200.build      # or __graft_entry__.build()

Output: paper_1803_03288_b200/libcommsched.so exporting only the cs_*
symbols of include/commsched.h (linker version script). CUDA runtime is
linked statically so the library only needs the driver at run time. Then
paper_1803_03288_b200/tictac_sched, the native sweep/bruteforce CLI over
the C ABI.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import site
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libcommsched.so")
CLI = os.path.join(PKG, "tictac_sched")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _cuda_home() -> str:
    for c in (os.environ.get("CUDA_HOME"), "/usr/local/cuda"):
        if c and os.path.exists(os.path.join(c, "bin", "nvcc")):
            return c
    nvcc = shutil.which("nvcc")
    if nvcc:
        return os.path.dirname(os.path.dirname(nvcc))
    raise RuntimeError("nvcc not found")


def _json_dir() -> str:
    cands = []
    for p in site.getsitepackages() + [site.getusersitepackages()]:
        cands.append(os.path.join(p, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
    for c in cands:
        if os.path.exists(os.path.join(c, "json.hpp")):
            return c
    raise RuntimeError("nlohmann/json.hpp (3.11.3) not found in site-packages")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    cuda = _cuda_home()
    nvcc = os.path.join(cuda, "bin", "nvcc")
    jdir = _json_dir()
    os.makedirs(OBJ, exist_ok=True)
    host = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    dev = sorted(glob.glob(os.path.join(CSRC, "device", "*.cu")))
    headers = (glob.glob(os.path.join(CSRC, "*", "*.h*")) + glob.glob(os.path.join(CSRC, "*", "*.cuh"))
               + [os.path.join(ROOT, "include", "commsched.h")])
    cxx = os.environ.get("CXX", "g++")
    jobs = []
    for src in host:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        cmd = [cxx, "-std=c++20", "-O2", "-fPIC", "-fvisibility=hidden", "-Wall", "-Wno-unused-function",
               f"-I{jdir}", f"-I{cuda}/include", f"-I{os.path.join(ROOT, 'include')}", "-c", src, "-o", obj]
        jobs.append((obj, [src] + headers, cmd))
    for src in dev:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        cmd = [nvcc, *ARCH, "-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden",
               "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills", f"-I{os.path.join(ROOT, 'include')}",
               "-c", src, "-o", obj]
        jobs.append((obj, [src] + headers, cmd))

    def run(job):
        obj, deps, cmd = job
        if not force and not _stale(obj, deps):
            return obj, ""
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return obj, r.stderr

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        results = list(ex.map(run, jobs))
    if verbose:
        for obj, msg in results:
            if msg.strip():
                print(f"[{os.path.basename(obj)}] {msg}", file=sys.stderr)
    objs = [o for o, _ in results]
    vers = os.path.join(OBJ, "exports.map")
    with open(vers, "w") as f:
        f.write("{ global: cs_*; local: *; };\n")
    if force or _stale(LIB, objs + [vers]):
        tmp = LIB + ".tmp"
        cmd = [nvcc, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
               "-Xlinker", f"--version-script={vers}", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    # the native batched CLI driver: a client of the C ABI only
    src = os.path.join(CSRC, "cli", "sched_main.cpp")
    if force or _stale(CLI, [src, LIB, os.path.join(ROOT, "include", "commsched.h")]):
        tmp = CLI + ".tmp"
        cmd = [cxx, "-std=c++20", "-O2", "-Wall", f"-I{jdir}", f"-I{os.path.join(ROOT, 'include')}", src,
               "-o", tmp, f"-L{PKG}", "-l:libcommsched.so", "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"CLI build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, CLI)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))

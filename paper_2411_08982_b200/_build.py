"""Build liblynx_b200.so in-tree for sm_100a (B200) with nvcc.

    python -m paper_2411_08982_b200._build        # or __graft_entry__.build()

Objects go to build/, the shared library to paper_2411_08982_b200/_lib/
(git-ignored, but shipped to the GPU box with the working tree).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIB_DIR, "liblynx_b200.so")

SOURCES = ["select.cu", "dispatch.cu", "ffn.cu", "attention.cu", "ep_p2p.cu", "capi.cu"]
HEADERS = ["ptx.cuh", "lynx_internal.cuh", "p2p.cuh", "npexp.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-diag-suppress", "550"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build liblynx_b200.so")


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, trace: bool = False, src_dir: str | None = None,
          out: str | None = None) -> str:
    """Compile liblynx_b200.so; trace=True builds the diagnostic variant
    liblynx_b200_trace.so (-DLYNX_TRACE: per-unit timeline records).
    src_dir/out build another source tree (A/B experiments) into `out`."""
    build_dir = os.path.join(BUILD, "trace") if trace else BUILD
    lib_path = LIB.replace(".so", "_trace.so") if trace else LIB
    extra = ["-DLYNX_TRACE"] if trace else []
    csrc, inc = CSRC, INCLUDE
    if src_dir is not None:
        csrc, inc = os.path.join(src_dir, "paper_2411_08982_b200", "csrc"), os.path.join(src_dir, "include")
        build_dir = os.path.join(BUILD, "ab_" + os.path.basename(out).replace(".so", "") + ("_t" if trace else ""))
        lib_path = out
    os.makedirs(build_dir, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    cc = nvcc()
    headers = [os.path.join(csrc, h) for h in HEADERS] + [os.path.join(inc, "lynx_b200.h")]
    objs, cmds = [], []
    for src in SOURCES:
        path = os.path.join(csrc, src)
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _newer(obj, [path] + headers):
            cmds.append([cc, *ARCH, *FLAGS, *extra, "-I", inc, "-c", path, "-o", obj])
    # translation units compile in parallel (one nvcc each)
    procs = []
    for cmd in cmds:
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd)))
    failed = [cmd for cmd, pr in procs if pr.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    if force or _newer(lib_path, objs):
        tmp = lib_path + ".tmp"
        cmd = [cc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-cudart", "static"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    if "--ab" in sys.argv:  # python -m paper_2411_08982_b200._build --ab <git-rev> <out.so>
        import tempfile
        rev, out = sys.argv[sys.argv.index("--ab") + 1], os.path.abspath(sys.argv[sys.argv.index("--ab") + 2])
        with tempfile.TemporaryDirectory() as tmp:
            subprocess.run(f"git -C {ROOT} archive {rev} paper_2411_08982_b200/csrc include | tar -x -C {tmp}",
                           shell=True, check=True)
            print(build(verbose=True, force=True, src_dir=tmp, out=out, trace="--trace" in sys.argv))
    else:
        print(build(verbose=True, force="--force" in sys.argv, trace="--trace" in sys.argv))

"""Build libhelios.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhelios.so")
DEBUG_LIB = os.path.join(HERE, "libhelios_debug.so")  # -DHELIOS_DEBUG: device invariant checks
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "--expt-relaxed-constexpr", f"-I{INCLUDE}"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return (_sources() + glob.glob(os.path.join(CSRC, "*.cuh")) +
            glob.glob(os.path.join(INCLUDE, "*.h")) + [os.path.abspath(__file__)])


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _deps())


def build_debug(force: bool = False) -> str:
    """libhelios_debug.so: the same sources with HELIOS_DEBUG (device-side
    HELIOS_DASSERT checks of the kernels' invariants: traversal stack depth,
    beam entry list bound, subray table index, waveform window, attribution);
    load it with HELIOS_LIB to run any test or tool under the checks."""
    if not force and os.path.exists(DEBUG_LIB):
        t = os.path.getmtime(DEBUG_LIB)
        if all(os.path.getmtime(p) <= t for p in _deps()):
            return DEBUG_LIB
    return build(force=True, defines=("HELIOS_DEBUG",), out=DEBUG_LIB)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile every csrc/*.cu for sm_100a and link libhelios.so (or `out`).
    `defines`: extra -D flags for experiment variants."""
    lib_path = out or LIB
    if not force and not defines and out is None and up_to_date():
        return LIB
    objdir = os.path.join(HERE, "build", "_".join(d.replace("=", "") for d in defines) or "default")
    os.makedirs(objdir, exist_ok=True)
    procs = []
    objs = []
    for src in _sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT, text=True)))
    failed = False
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed building libhelios (see output above)")
    tmp = lib_path + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", *objs, "-o", tmp])
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    if "--debug" in sys.argv:
        print(build_debug(force="--force" in sys.argv))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                    out=outs[0] if outs else None))

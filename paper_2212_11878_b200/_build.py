"""Build libmpcd.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext).

-fmad=false / -ffp-contract=off are part of the numerics contract: the
reference never fuses a*b+c.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libmpcd.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
    deps += glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, defines=None, out: str | None = None) -> str:
    """Compile libmpcd.so (or a tuning variant with -D`defines` into `out`).

    Each translation unit (the engine, the scan, the stage kernels and the
    four step-mode variant units) compiles in its own nvcc process, in
    parallel; the objects are then linked into the shared library."""
    import concurrent.futures as cf
    import tempfile

    target = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    flags = [f"-D{d}" for d in (defines or [])]
    # tuning builds only: extra nvcc flags (e.g. ptxas options) from the environment
    flags += os.environ.get("MPCD_NVCC_EXTRA", "").split()
    base = [nvcc()]
    # the distro g++ is the host compiler nvcc 12.9 supports here
    if os.path.exists("/usr/bin/g++"):
        base += ["-ccbin", "/usr/bin/g++"]
    with tempfile.TemporaryDirectory(prefix="mpcd_build_") as tmp:
        jobs = []
        for src in sources():
            obj = os.path.join(tmp, os.path.basename(src)[:-3] + ".o")
            jobs.append((obj, [*base, *NVCC_FLAGS, *flags, "-I", INCLUDE, "-I", CSRC,
                               "-c", "-o", obj, src]))
        if verbose:
            for _, cmd in jobs:
                print(" ".join(cmd))

        def run(cmd):
            return subprocess.run(cmd, capture_output=True, text=True)

        with cf.ThreadPoolExecutor(max_workers=len(jobs)) as ex:
            results = list(ex.map(run, [cmd for _, cmd in jobs]))
        for (_, cmd), r in zip(jobs, results):
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}{r.stderr}")
            if verbose and (r.stdout or r.stderr):
                print(r.stdout + r.stderr)
        link = [*base, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                "-o", target + ".tmp", *[obj for obj, _ in jobs]]
        if verbose:
            print(" ".join(link))
        subprocess.run(link, check=True)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))

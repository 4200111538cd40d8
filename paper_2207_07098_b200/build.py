"""Build libsemflow_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2207_07098_b200.build [--force]

The shared object is written next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsemflow_b200.so")
# the checked build: device bounds checks (SF_CHECK in csrc/common.cuh) compiled in
OUT_CHECKED = os.path.join(HERE, "libsemflow_b200_checked.so")
ROOT = os.path.dirname(HERE)

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC",
    "-I", os.path.join(ROOT, "include"),
]
OBJDIR = os.path.join(ROOT, "build", "obj")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(out=OUT):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh"))
    deps.append(os.path.join(ROOT, "include", "semflow_b200.h"))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False, checked=False):
    out = OUT_CHECKED if checked else OUT
    if not force and not _stale(out):
        return out
    from concurrent.futures import ThreadPoolExecutor

    nvcc = os.environ.get("NVCC", "nvcc")
    objdir = OBJDIR + ("_checked" if checked else "")
    os.makedirs(objdir, exist_ok=True)
    flags = NVCC_FLAGS + (["-DSF_CHECKS"] if checked else [])
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        jobs.append((obj, [nvcc, *flags, "-c", src, "-o", obj]))

    def run(job):
        if verbose:
            print(" ".join(job[1]), flush=True)
        subprocess.run(job[1], check=True)
        return job[0]

    with ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
        objs = list(ex.map(run, jobs))
    subprocess.run([nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-o", out + ".tmp", *objs], check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))

"""Compile csrc/*.cu into paper_2510_03557_b200/libhb.so for sm_100a (in-tree,
so the .so travels to the GPU box with the repo snapshot)."""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libhb.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--extended-lambda", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "-diag-suppress", "177"]
SOURCES = ["hb_sort.cu", "hb_mesh.cu", "hb_pairs.cu", "hb_crk.cu", "hb_step.cu", "hb_sph.cu", "hb_halo.cu", "hb_grav2.cu", "hb_pm.cu", "hb_fof.cu", "hb_crc.cu", "hb_levels.cu"]


def _compile(src: str, obj: str) -> None:
    cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")


def build(verbose: bool = False) -> str:
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    srcs = [s for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    objs = [os.path.join(objdir, s.replace(".cu", ".o")) for s in srcs]
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(HERE, "..", "include", "hb.h")]
    newest_dep = max(os.path.getmtime(d) for d in deps)
    todo = [(s, o) for s, o in zip(srcs, objs)
            if not os.path.exists(o) or os.path.getmtime(o) < newest_dep]
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        list(ex.map(lambda so: _compile(*so), todo))
    if todo or not os.path.exists(OUT):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    if verbose:
        print(f"built {OUT}")
    return OUT


if __name__ == "__main__":
    build(verbose=True)

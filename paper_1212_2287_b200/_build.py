"""Build the native library in-tree: ``paper_1212_2287_b200/_ts_gpu.so``.

One nvcc invocation compiles the CUDA kernels for sm_100a only and the host
C++ (packer + C ABI) into a single shared object with a plain C ABI
(``include/treescore_gpu.h``).  No ``--use_fast_math``: the traversal's
``x >= theta`` must see denormals (no FTZ) and the f64 leaf sum must stay
multiply-then-add.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.environ.get("TS_GPU_SO") or os.path.join(HERE, "_ts_gpu.so")
SOURCES = ["ts_kernels.cu", "ts_stream.cu", "ts_stream_i0.cu", "ts_stream_i1.cu",
           "ts_stream_i2.cu", "ts_stream_i3.cu", "ts_stream_i4.cu", "ts_cstream.cu", "ts_cstream_w8.cu", "ts_cstream_w16.cu", "ts_trace.cu", "ts_synth.cu", "ts_rank.cu", "ts_rank_i0.cu", "ts_rank_i1.cu", "ts_rank_i2.cu",
           "ts_pack.cpp", "ts_parse.cpp", "ts_capi.cpp", "ts_nccl.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, s) for s in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "treescore_gpu.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile each translation unit in parallel, then link one .so."""
    if not force and not _stale():
        return SO
    from concurrent.futures import ThreadPoolExecutor
    import tempfile
    objdir = os.path.join(tempfile.gettempdir(), "ts_gpu_build", os.path.basename(SO))
    os.makedirs(objdir, exist_ok=True)
    common = [nvcc(), *ARCH, *os.environ.get("TS_NVCC_EXTRA", "").split(), "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
              "-Xptxas", "-warn-spills"]
    if verbose:
        common += ["-Xptxas", "-v"]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = common + ["-c", os.path.join(CSRC, src), "-o", obj]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, cmd, res

    with ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, SOURCES))
    for src, _obj, cmd, res in results:
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src} ({res.returncode}):\n{' '.join(cmd)}\n"
                               f"{res.stdout}\n{res.stderr}")
        if verbose:
            sys.stderr.write(res.stderr)
    link = [nvcc(), *ARCH, "-shared", "-o", SO + ".tmp"] + [r[1] for r in results] + ["-ldl"]
    res = subprocess.run(link, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{' '.join(link)}\n{res.stdout}\n{res.stderr}")
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

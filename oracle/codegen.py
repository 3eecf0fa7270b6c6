"""CPU CodeGen baseline -- TEST / BASELINE INFRASTRUCTURE ONLY.

A restatement of the reference's *generated* strategy
(``pkg/src/treescore/codegen.py``), used as the second CPU baseline that
SURVEY section 8(d)(ii) asks for beside the VPred port: the faster of the two
is the reported CPU number.  Only ``tests/``, ``tools/`` and ``bench.py``'s
CPU legs use it; the product package never imports it.

What the reference does, and what this file restates:

* ``emit_source`` (ref ``codegen.py:89-122``): one ``static float tree_<k>``
  per tree as a nested if/else -- ``if (x[fid] < thr) { left } else { right }``
  (strict ``<`` goes left: the shared tie rule, ``x >= thr`` goes right) --
  returning the leaf as a float; ``double score_ensemble(const float *x)``
  adds ``acc += w * (double) tree_k(x)`` in tree order from ``acc = 0.0``;
  ``void score_batch(const float *x, int64_t n, int64_t f, double *out)``
  applies it row by row.  Constants are C99 hex-float literals (exact; ref
  ``codegen.py:67-72``).  This emitter walks the FLAT arrays (no Python
  ``Node`` objects), with an explicit stack instead of recursion, and emits
  the same C text shape.
* ``compile_unit`` (ref ``codegen.py:189-223``): ``cc -O3
  -fomit-frame-pointer -pipe -shared -fPIC`` (ref ``OPT_FLAGS``,
  ``codegen.py:40``), then ``ctypes`` loads ``score_batch``.  No ``-march``:
  the x86-64 baseline has no FMA, so ``acc += w * t`` is never contracted
  (bit-identical to the f64 tree-order sum of the other strategies).
* Multi-core timing as SURVEY 8(d)(ii) specifies: one thread per core over
  row shards through ``score_batch`` (ctypes releases the GIL during the
  foreign call, as the reference's ``GeneratedUnit.score_batch_into`` does).
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
import threading
import time

import numpy as np

OPT_FLAGS = ("-O3", "-fomit-frame-pointer", "-pipe")   # ref codegen.py:40
_HERE = os.path.dirname(os.path.abspath(__file__))
GEN_DIR = os.path.join(_HERE, "_gen")


def _c_float(v) -> str:
    return float.hex(float(np.float32(v))) + "f"


def _c_double(v) -> str:
    return float.hex(float(v))


def emit_source(flat) -> str:
    """C source of the reference's generated scorer for a flat ensemble
    (``paper_1212_2287_b200.model.FlatModel`` or its ``arrays()`` tuple plus
    ``num_features``)."""
    F = int(flat.num_features)
    off, w, fid, val, left, right = flat.arrays()
    T = len(off) - 1
    out = ["/* Generated tree-ensemble scorer. Do not edit. */",
           f"/* trees={T} num_features={F} */",
           "#include <stdint.h>", ""]
    a = out.append
    for k in range(T):
        base = int(off[k])
        a(f"static float tree_{k}(const float *x) {{")
        # explicit stack of (node, indent, phase); phase 0 = open, 1 = else, 2 = close
        stack = [(0, 1, 0)]
        while stack:
            node, ind, ph = stack.pop()
            pad = "    " * ind
            g = base + node
            if ph == 0:
                if fid[g] < 0:
                    a(f"{pad}return {_c_float(val[g])};")
                    continue
                a(f"{pad}if (x[{int(fid[g])}] < {_c_float(val[g])}) {{")
                stack.append((node, ind, 1))
                stack.append((int(left[g]), ind + 1, 0))
            elif ph == 1:
                a(f"{pad}}} else {{")
                stack.append((node, ind, 2))
                stack.append((int(right[g]), ind + 1, 0))
            else:
                a(f"{pad}}}")
        a("}")
        a("")
    a("double score_ensemble(const float *x) {")
    a("    double acc = 0.0;")
    for k in range(T):
        a(f"    acc += {_c_double(w[k])} * (double) tree_{k}(x);")
    a("    return acc;")
    a("}")
    a("")
    a("void score_batch(const float *x, int64_t n, int64_t f, double *out) {")
    a("    int64_t i;")
    a("    for (i = 0; i < n; i++) {")
    a("        out[i] = score_ensemble(x + i * f);")
    a("    }")
    a("}")
    return "\n".join(out) + "\n"


class GeneratedUnit:
    """A compiled generated scorer (ref ``GeneratedUnit``, codegen.py:125-178)."""

    def __init__(self, so_path: str, compile_s: float = 0.0):
        self.path = so_path
        self.compile_s = compile_s
        self._lib = ctypes.CDLL(so_path)
        self._batch = self._lib.score_batch
        self._batch.restype = None
        self._batch.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]

    def score_batch_into(self, x: np.ndarray, out: np.ndarray) -> None:
        assert x.dtype == np.float32 and x.flags.c_contiguous and out.dtype == np.float64
        self._batch(x.ctypes.data, x.shape[0], x.shape[1], out.ctypes.data)

    def score(self, x: np.ndarray, threads: int = 1) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty(x.shape[0], np.float64)
        self.score_parallel(x, out, threads)
        return out

    def score_parallel(self, x: np.ndarray, out: np.ndarray, threads: int) -> None:
        """One thread per core over contiguous row shards (GIL released in C)."""
        n = x.shape[0]
        threads = max(1, min(threads, n))
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        ts = [threading.Thread(target=self.score_batch_into,
                               args=(x[bounds[i]:bounds[i + 1]], out[bounds[i]:bounds[i + 1]]))
              for i in range(threads) if bounds[i + 1] > bounds[i]]
        for t in ts:
            t.start()
        for t in ts:
            t.join()


def model_key(flat) -> str:
    h = hashlib.sha1()
    for arr in flat.arrays():
        h.update(np.ascontiguousarray(arr).tobytes())
    h.update(str(int(flat.num_features)).encode())
    return h.hexdigest()[:16]


def compile_unit(flat, cc: str = "gcc", cache: bool = True) -> GeneratedUnit:
    """Emit, compile (``cc -O3 -fomit-frame-pointer -pipe``) and load; the
    shared object is cached under ``oracle/_gen/<model hash>.so`` so a
    build-time compile (``__graft_entry__.build``) travels to the GPU box."""
    os.makedirs(GEN_DIR, exist_ok=True)
    key = model_key(flat)
    so = os.path.join(GEN_DIR, f"{key}.so")
    if cache and os.path.exists(so):
        return GeneratedUnit(so)
    src = os.path.join(GEN_DIR, f"{key}.c")
    with open(src, "w") as fh:
        fh.write(emit_source(flat))
    t0 = time.time()
    tmp = so + f".tmp{os.getpid()}"
    proc = subprocess.run([cc, *OPT_FLAGS, "-shared", "-fPIC", "-o", tmp, src],
                          capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"compiler failed (exit {proc.returncode}):\n{proc.stderr or proc.stdout}")
    os.replace(tmp, so)
    os.remove(src)
    return GeneratedUnit(so, time.time() - t0)


def cached_unit(flat):
    """The prebuilt unit for ``flat`` if ``compile_unit`` already made it, else None."""
    so = os.path.join(GEN_DIR, f"{model_key(flat)}.so")
    return GeneratedUnit(so) if os.path.exists(so) else None

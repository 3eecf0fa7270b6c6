"""GPU evaluator: the reference's ``Evaluator`` interface over the C ABI.

Mirrors ref ``treescore/evaluators.py``:

* ``build(ensemble, kind, batch_size=None)`` (ref :565-585) -- accepts the
  reference's kind names with its argument checks and serves them all with
  the GPU evaluator; ``build_gpu`` is the direct constructor, the way the
  reference builds its native strategy through ``build_generated``
  (ref codegen.py:247-253).
* ``Evaluator.predict(x)`` / ``predict_batch(data)`` / ``_predict_into``
  (ref :187-231) with the same ``ValueError`` messages for shape mismatch
  (ref :204-220); ``stored_node_count`` (ref :197-200) counts complete-table
  entries like the predicated kinds (ref :548-550).
* ``leaf_indices(data)`` returns the per-tree predicated leaf ordinals --
  what ``batch_kernel`` / ``leaf_index_predicated`` compute per tree
  (ref :90-99, :122-134).

Host side is PyTorch (device buffers, the current CUDA stream); all scoring
runs in ``_ts_gpu.so``.  Inputs may be a ``Dataset``, anything numpy can view
as float32, or a torch tensor on the CPU or on the evaluator's GPU.
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib
from .data import Dataset
from .model import DepthLimitError, Ensemble, FlatModel, ModelSemanticError


class StrategyKind(enum.Enum):
    """The reference's strategy names (ref evaluators.py:56-68) plus the GPU
    one.  Every strategy scores bit-identically by the reference's contract,
    so ``build`` serves all accepted kinds with the GPU evaluator; the kind
    only selects the reference's argument checks."""

    HEAP_LINKED = "heap_linked"
    COMPACT_LINKED = "compact_linked"
    CONTIGUOUS = "contiguous"
    PREDICATED = "predicated"
    VPREDICATED = "vpredicated"
    GENERATED = "generated"
    GPU_VPREDICATED = "gpu_vpredicated"

    def __str__(self):
        return self.value


ALL_STRATEGIES = tuple(StrategyKind)  # ref evaluators.py:69
_LINKED_KINDS = (StrategyKind.HEAP_LINKED, StrategyKind.COMPACT_LINKED, StrategyKind.CONTIGUOUS)


def _torch():
    import torch
    return torch


def _ptr(a) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


@dataclass(frozen=True)
class TracedPrediction:
    """ref evaluators.py:592-596: score, union of path feature ids, logical
    left-to-right leaf ordinal per tree."""

    score: float
    visited_features: frozenset
    visited_leaves: tuple


@dataclass(frozen=True)
class CoverageReport:
    """ref bench.py:153-158: fraction of the feature space examined per
    prediction (mean and population variance over instances)."""

    mean_fraction: float
    variance: float
    num_instances: int


class GpuModel:
    """Packed device tables of one ensemble on one GPU (``ts_pack``)."""

    def __init__(self, model, device: int | None = None, trace: bool = False,
                 any_depth: bool = False, rank: bool = True):
        torch = _torch()
        if not torch.cuda.is_available():
            raise _lib.NativeLibraryError("no CUDA device: the GPU scorer has no CPU fallback")
        lib = _lib.load()
        flat = model.flat() if isinstance(model, Ensemble) else model
        if not isinstance(flat, FlatModel):
            raise TypeError("model must be an Ensemble or a FlatModel")
        self.device = torch.cuda.current_device() if device is None else int(device)
        arrs = [np.ascontiguousarray(flat.tree_off, np.int64),
                np.ascontiguousarray(flat.weight, np.float64),
                np.ascontiguousarray(flat.fid, np.int32),
                np.ascontiguousarray(flat.value, np.float32),
                np.ascontiguousarray(flat.left, np.int32),
                np.ascontiguousarray(flat.right, np.int32)]
        desc = _lib.ModelDesc(int(flat.num_features), int(flat.num_trees),
                              *[a.ctypes.data for a in arrs])
        handle = ctypes.c_void_p()
        # rank=False keeps deep complete trees in the fp32 layout (the fused
        # cross-GPU pipeline, score_pipe, runs on that layout only)
        flags = ((_lib.TS_PACK_TRACE if trace else 0) | (_lib.TS_PACK_ANY_DEPTH if any_depth else 0)
                 | (0 if rank else _lib.TS_PACK_NO_RANK))
        rc = lib.ts_pack_ex(ctypes.byref(desc), self.device, flags,
                            ctypes.byref(handle))
        if rc == _lib.TS_ERR_DEPTH:
            raise DepthLimitError(_lib.last_error())
        if rc == _lib.TS_ERR_INVALID:
            raise ModelSemanticError(_lib.last_error())
        if rc != _lib.TS_OK:
            raise RuntimeError(f"ts_pack failed ({rc}): {_lib.last_error()}")
        self._lib = lib
        self.handle = handle
        info = _lib.ModelInfo()
        lib.ts_model_get_info(handle, ctypes.byref(info))
        self.info = info.as_dict()
        self.num_features = int(flat.num_features)
        self.num_trees = int(flat.num_trees)
        self.node_count = int(flat.tree_off[-1])  # logical nodes (internal + leaves)

    def _check_x(self, x, what="x"):
        torch = _torch()
        if x.dim() != 2 or x.dtype != torch.float32 or not x.is_cuda:
            raise TypeError(f"{what} must be a 2-D float32 CUDA tensor")
        if x.stride(1) != 1:
            raise ValueError(f"{what} rows must be contiguous (stride(1) == 1)")
        if x.device.index != self.device:
            # the kernel runs on the model's GPU: another GPU's pointer would
            # fault there (no peer mapping) and poison the whole context
            raise ValueError(f"{what} is on cuda:{x.device.index}, the model on cuda:{self.device}")

    def _check_buf(self, t, what, dtype, n):
        """Device buffers the kernel writes: right dtype, device, contiguity
        and at least ``n`` elements (a short or mistyped buffer would be
        overrun on the device)."""
        if t is None:
            return
        if not t.is_cuda or t.device.index != self.device:
            raise ValueError(f"{what} must be a CUDA tensor on cuda:{self.device}")
        if t.dtype != dtype:
            raise ValueError(f"{what} must have dtype {dtype}, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{what} must be contiguous")
        if t.numel() < n:
            raise ValueError(f"{what} has {t.numel()} elements, needs >= {n}")

    def score(self, x, out=None, ordinals=None, status=None, stream=None, accumulate=False):
        """Enqueue scoring of a CUDA float32 ``[n, f]`` tensor (row stride >= f).

        ``out``: f64 CUDA tensor ``[n]`` (allocated if None).  ``ordinals``:
        optional uint16-compatible CUDA tensor ``[T, >= n]`` (torch.int16 or
        torch.uint16) receiving predicated leaf ordinals.  ``status``: optional
        int32 CUDA scalar OR-ed with 1 on non-finite input.  Returns ``out``.
        Stream-ordered on ``stream`` (default: torch's current stream).
        ``accumulate``: ``out`` holds the partial sum of the preceding trees
        (a tree shard); scoring continues from it (``ts_score_ex``).
        """
        torch = _torch()
        self._check_x(x)
        n, f = x.shape
        if f != self.num_features:
            raise ValueError(f"dataset has shape {tuple(x.shape)}, expected (n, {self.num_features})")
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=x.device)
        self._check_buf(out, "out", torch.float64, n)
        self._check_buf(status, "status", torch.int32, 1)
        ld_ord = 0
        ord_ptr = None
        if ordinals is not None:
            if ordinals.element_size() != 2 or ordinals.dim() != 2 or ordinals.stride(1) != 1 \
                    or ordinals.shape[0] != self.num_trees or ordinals.shape[1] < n \
                    or ordinals.is_floating_point():
                raise ValueError("ordinals must be a [T, >=n] 16-bit integer row-major tensor")
            if not ordinals.is_cuda or ordinals.device.index != self.device:
                raise ValueError(f"ordinals must be a CUDA tensor on cuda:{self.device}")
            ld_ord = ordinals.stride(0)
            ord_ptr = ctypes.c_void_p(ordinals.data_ptr())
        if stream is None:
            stream = torch.cuda.current_stream(x.device)
        ld = x.stride(0) if n > 1 else f   # size-1 leading dims may carry stride 0
        rc = self._lib.ts_score_ex(self.handle, ctypes.c_void_p(x.data_ptr()), n, f, ld,
                                   ctypes.c_void_p(out.data_ptr()), ord_ptr, ld_ord,
                                   ctypes.c_void_p(status.data_ptr()) if status is not None
                                   else None, 1 if accumulate else 0,
                                   ctypes.c_void_p(stream.cuda_stream))
        if rc == _lib.TS_ERR_DEPTH:
            raise DepthLimitError(_lib.last_error())
        if rc != _lib.TS_OK:
            raise RuntimeError(f"ts_score failed ({rc}): {_lib.last_error()}")
        return out

    def score_pipe(self, x, out=None, sums_in=0, flags_in=0, sums_out=0, flags_out=0,
                   epoch=1, stream=None):
        """``ts_score_pipe``: one stage of the fused cross-GPU running-sum pipeline.

        ``sums_in``/``flags_in``: this rank's :class:`PipeBuffers` (0 on the
        first rank); ``sums_out``/``flags_out``: the next rank's buffers as
        device pointers (:class:`PeerBuffers`, 0 on the last rank, which
        writes ``out``).  ``epoch`` must grow by one per call.
        """
        torch = _torch()
        self._check_x(x)
        n, f = x.shape
        if f != self.num_features:
            raise ValueError(f"dataset has shape {tuple(x.shape)}, expected (n, {self.num_features})")
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=x.device)
        self._check_buf(out, "out", torch.float64, n)
        if stream is None:
            stream = torch.cuda.current_stream(x.device)
        pipe = _lib.Pipe(sums_in or None, flags_in or None, sums_out or None, flags_out or None,
                         int(epoch) & 0xFFFFFFFF)
        ld = x.stride(0) if n > 1 else f
        rc = self._lib.ts_score_pipe(self.handle, ctypes.c_void_p(x.data_ptr()), n, f, ld,
                                     ctypes.c_void_p(out.data_ptr()), ctypes.byref(pipe),
                                     ctypes.c_void_p(stream.cuda_stream))
        if rc != _lib.TS_OK:
            raise RuntimeError(f"ts_score_pipe failed ({rc}): {_lib.last_error()}")
        return out

    def trace(self, x, out=None, leaf_ord=None, visited=None, stream=None):
        """``ts_trace`` on a CUDA float32 ``[n, f]`` tensor (model packed with trace=True)."""
        torch = _torch()
        self._check_x(x)
        n, f = x.shape
        if f != self.num_features:
            raise ValueError(f"dataset has shape {tuple(x.shape)}, expected (n, {self.num_features})")
        words = (self.num_features + 31) // 32
        self._check_buf(out, "out", torch.float64, n)
        self._check_buf(visited, "visited", torch.int32, n * words)
        if leaf_ord is not None:
            if leaf_ord.element_size() != 2 or leaf_ord.dim() != 2 or leaf_ord.stride(1) != 1 \
                    or leaf_ord.shape[0] != self.num_trees or leaf_ord.shape[1] < n:
                raise ValueError("leaf_ord must be a [T, >=n] 16-bit row-major tensor")
            if not leaf_ord.is_cuda or leaf_ord.device.index != self.device:
                raise ValueError(f"leaf_ord must be a CUDA tensor on cuda:{self.device}")
        if stream is None:
            stream = torch.cuda.current_stream(x.device)
        p = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
        ld = x.stride(0) if n > 1 else f
        rc = self._lib.ts_trace(self.handle, p(x), n, f, ld, p(out), p(leaf_ord),
                                leaf_ord.stride(0) if leaf_ord is not None else 0, p(visited),
                                words, ctypes.c_void_p(stream.cuda_stream))
        if rc != _lib.TS_OK:
            raise RuntimeError(f"ts_trace failed ({rc}): {_lib.last_error()}")

    def score_host(self, matrix: np.ndarray, out: np.ndarray) -> None:
        """``ts_score_host``: host fp32 ``[n, f]`` -> host f64 ``[n]``."""
        rc = self._lib.ts_score_host(self.handle, _ptr(matrix), matrix.shape[0],
                                     matrix.shape[1], _ptr(out))
        if rc == _lib.TS_ERR_NONFINITE:
            raise ValueError("dataset contains non-finite values")
        if rc == _lib.TS_ERR_SHAPE:
            raise ValueError(_lib.last_error())
        if rc != _lib.TS_OK:
            raise RuntimeError(f"ts_score_host failed ({rc}): {_lib.last_error()}")

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self._lib.ts_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


class PipeBuffers:
    """This rank's receive side of the fused pipeline (``ts_pipe_alloc``):
    f64 ``sums[n]`` and zeroed u32 ``flags[ceil(n/32)]`` plus 64-byte CUDA IPC
    handles the previous rank opens with :class:`PeerBuffers`."""

    def __init__(self, n: int, device: int):
        self._lib = lib = _lib.load()
        s, f = ctypes.c_void_p(), ctypes.c_void_p()
        hs, hf = ctypes.create_string_buffer(64), ctypes.create_string_buffer(64)
        rc = lib.ts_pipe_alloc(int(device), int(n), ctypes.byref(s), ctypes.byref(f), hs, hf)
        if rc != _lib.TS_OK:
            raise RuntimeError(f"ts_pipe_alloc failed ({rc}): {_lib.last_error()}")
        self.sums, self.flags = s.value, f.value
        self.handles = (hs.raw, hf.raw)

    def close(self):
        if getattr(self, "sums", None):
            self._lib.ts_pipe_free(self.sums, self.flags)
            self.sums = self.flags = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


class PeerBuffers:
    """Another process's :class:`PipeBuffers` mapped here (``ts_ipc_open``)."""

    def __init__(self, handles):
        self._lib = lib = _lib.load()
        ptrs = []
        for h in handles:
            p = ctypes.c_void_p()
            rc = lib.ts_ipc_open(ctypes.create_string_buffer(bytes(h), 64), ctypes.byref(p))
            if rc != _lib.TS_OK:
                for q in ptrs:
                    lib.ts_ipc_close(q)
                raise RuntimeError(f"ts_ipc_open failed ({rc}): {_lib.last_error()}")
            ptrs.append(p.value)
        self.sums, self.flags = ptrs

    def close(self):
        if getattr(self, "sums", None):
            self._lib.ts_ipc_close(self.sums)
            self._lib.ts_ipc_close(self.flags)
            self.sums = self.flags = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


class GpuEvaluator:
    """Immutable GPU scoring strategy built from an ensemble.

    ``predict`` / ``predict_batch`` return exactly the reference's f64 scores
    (bit-identical: same tie rule, dummy routing, fp32 tables, f64 tree-order
    multiply-then-add).  Non-finite inputs raise ``ValueError`` (the
    reference's ``Dataset`` contract, ref data.py:50-51); there is no silent
    NaN routing.
    """

    kind = StrategyKind.GPU_VPREDICATED

    def __init__(self, ensemble, batch_size: int | None = None, device: int | None = None,
                 trace: bool = False, kind: StrategyKind | None = None):
        if kind is not None:
            self.kind = StrategyKind(kind)
        if batch_size is not None:
            batch_size = int(batch_size)
            if batch_size < 1:
                raise ValueError(f"batch_size must be >= 1, got {batch_size}")
        self.batch_size = batch_size
        # the reference's linked kinds walk trees of any depth (no complete
        # table); so does the GPU packer's child-index layout
        self.model = GpuModel(ensemble, device, trace=trace,
                              any_depth=self.kind in _LINKED_KINDS)
        self.num_features = self.model.num_features
        self.num_trees = self.model.num_trees
        self.device = self.model.device

    # -- reference-compatible surface ---------------------------------------------

    def predict(self, x) -> float:
        x = np.ascontiguousarray(x, dtype=np.float32)
        if x.ndim != 1 or x.shape[0] != self.num_features:
            raise ValueError(f"feature vector has shape {x.shape}, expected ({self.num_features},)")
        return float(self.predict_batch(x[None, :])[0])

    def predict_batch(self, data) -> np.ndarray:
        torch = _torch()
        if isinstance(data, torch.Tensor):
            return self._predict_tensor(data).cpu().numpy()
        matrix = self._coerce_matrix(data)
        out = np.empty(matrix.shape[0], dtype=np.float64)
        self._predict_into(matrix, out)
        return out

    def _predict_into(self, matrix, out) -> None:
        if matrix.shape[0] == 0:
            return
        if out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float64 array")
        self.model.score_host(np.ascontiguousarray(matrix, dtype=np.float32), out)

    def _coerce_matrix(self, data) -> np.ndarray:
        matrix = data.matrix if isinstance(data, Dataset) else np.ascontiguousarray(
            data, dtype=np.float32)
        if matrix.ndim != 2 or matrix.shape[1] != self.num_features:
            raise ValueError(f"dataset has shape {matrix.shape}, expected (n, {self.num_features})")
        return matrix

    @property
    def stored_node_count(self) -> int:
        """As the reference's kind would count it (ref evaluators.py:297-474):
        the trees' own nodes for the linked / contiguous kinds, complete-table
        slots (2^(d+1) - 1 per tree) for the predicated ones."""
        if self.kind in _LINKED_KINDS:
            return self.model.node_count
        return int(self.model.info["table_entries"])

    # -- GPU-native extras ---------------------------------------------------------

    def _predict_tensor(self, x):
        torch = _torch()
        if x.dim() != 2 or x.shape[1] != self.num_features:
            raise ValueError(f"dataset has shape {tuple(x.shape)}, expected (n, {self.num_features})")
        dev = torch.device("cuda", self.device)
        x = x.to(device=dev, dtype=torch.float32)
        if x.stride(1) != 1:
            x = x.contiguous()
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        out = self.model.score(x, status=status)
        if int(status.item()):
            raise ValueError("dataset contains non-finite values")
        return out

    def score_device(self, x, out=None, stream=None):
        """Scores of a resident CUDA tensor, stream-ordered, no host sync."""
        return self.model.score(x, out=out, stream=stream)

    def leaf_indices(self, data) -> np.ndarray:
        """Per-tree predicated leaf ordinals, shape ``(T, n)``, int64.

        Row ``t`` equals the reference ``batch_kernel(d_t)`` result on
        ``expand_to_complete(tree_t)`` (ref evaluators.py:90-99).
        """
        torch = _torch()
        dev = torch.device("cuda", self.device)
        if isinstance(data, torch.Tensor):
            x = data.to(device=dev, dtype=torch.float32).contiguous()
        else:
            x = torch.from_numpy(self._coerce_matrix(data)).to(dev)
        n = x.shape[0]
        ords = torch.empty((self.num_trees, max(n, 1)), dtype=torch.int16, device=dev)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        if n:
            self.model.score(x, ordinals=ords, status=status)
        if int(status.item()):
            raise ValueError("dataset contains non-finite values")
        return ords[:, :n].cpu().numpy().view(np.uint16).astype(np.int64)

    # -- input pipeline ---------------------------------------

    def predict_fvec(self, path, chunk_rows: int = 1 << 18) -> np.ndarray:
        """Score an FVEC file (ref data.py:72-96) of any size, streaming it.

        A reader thread fills one pinned host buffer from disk while the GPU
        scores the other (``ts_score_host``: chunked H2D overlapped with the
        kernels, ctypes releases the GIL), so file IO, PCIe and compute
        overlap and N is not bounded by HBM.  Non-finite values raise
        ``ValueError`` like ``read_fvec``.
        """
        import threading

        from .data import fvec_header, read_fvec_into
        torch = _torch()
        count, f, _off = fvec_header(path)
        if f != self.num_features:
            raise ValueError(f"dataset has shape ({count}, {f}), expected (n, {self.num_features})")
        out = np.empty(count, dtype=np.float64)
        if count == 0:
            return out
        rows = max(1, min(chunk_rows, count))
        bufs = [torch.empty((rows, f), dtype=torch.float32, pin_memory=True).numpy()
                for _ in range(2)]
        filled = [threading.Semaphore(0), threading.Semaphore(0)]
        free = [threading.Semaphore(1), threading.Semaphore(1)]
        got = [0, 0]
        err = []
        stop = threading.Event()

        def reader():
            try:
                k = 0
                for r0 in range(0, count, rows):
                    free[k].acquire()
                    if stop.is_set():
                        return
                    got[k] = read_fvec_into(path, bufs[k], r0)
                    filled[k].release()
                    k ^= 1
            except Exception as exc:  # noqa: BLE001 - re-raised on the caller's thread
                err.append(exc)
                for sem in filled:
                    sem.release()

        th = threading.Thread(target=reader, daemon=True)
        th.start()
        k = 0
        try:
            for r0 in range(0, count, rows):
                filled[k].acquire()
                if err:
                    raise err[0]
                m = got[k]
                self.model.score_host(bufs[k][:m], out[r0:r0 + m])
                free[k].release()
                k ^= 1
        finally:
            stop.set()
            for sem in free:
                sem.release()
            th.join(timeout=60)
        return out

    # -- traced prediction (ref evaluators.py:599-620, bench.py:412-427) ---------

    def trace_batch(self, data):
        """``(scores f64[n], visited uint32[n, ceil(F/32)], leaves int64[T, n])``:
        per-instance visited-feature bitsets and logical leaf ordinals."""
        torch = _torch()
        dev = torch.device("cuda", self.device)
        if isinstance(data, torch.Tensor):
            x = data.to(device=dev, dtype=torch.float32).contiguous()
        else:
            x = torch.from_numpy(self._coerce_matrix(data)).to(dev)
        n = x.shape[0]
        words = (self.num_features + 31) // 32
        out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
        vis = torch.zeros((max(n, 1), words), dtype=torch.int32, device=dev)
        ords = torch.empty((self.num_trees, max(n, 1)), dtype=torch.int16, device=dev)
        if n:
            self.model.trace(x, out=out, leaf_ord=ords, visited=vis)
        return (out[:n].cpu().numpy(), vis[:n].cpu().numpy().view(np.uint32),
                ords[:, :n].cpu().numpy().view(np.uint16).astype(np.int64))

    def predict_traced(self, x) -> TracedPrediction:
        x = np.ascontiguousarray(x, dtype=np.float32)
        if x.ndim != 1 or x.shape[0] != self.num_features:
            raise ValueError(f"feature vector has shape {x.shape}, expected ({self.num_features},)")
        s, vis, leaves = self.trace_batch(x[None, :])
        bits = np.unpackbits(vis[0].view(np.uint8), bitorder="little")[:self.num_features]
        return TracedPrediction(float(s[0]), frozenset(np.flatnonzero(bits).tolist()),
                                tuple(int(v) for v in leaves[:, 0]))

    def feature_coverage(self, data) -> CoverageReport:
        """Mean fraction of features examined per instance (ref bench.py:412-427)."""
        matrix = data.matrix if isinstance(data, Dataset) else self._coerce_matrix(data)
        n = matrix.shape[0]
        if n == 0:
            return CoverageReport(0.0, 0.0, 0)
        _s, vis, _l = self.trace_batch(matrix)
        counts = np.unpackbits(vis.view(np.uint8), axis=1, bitorder="little").sum(axis=1)
        fractions = counts.astype(np.float64) / self.num_features
        return CoverageReport(float(fractions.mean()), float(fractions.var()), n)

    def close(self):
        self.model.close()

    def __repr__(self):
        return f"GpuEvaluator(kind={self.kind}, trees={self.num_trees}, device={self.device})"


def build_gpu(ensemble, batch_size: int | None = None, device: int | None = None,
              trace: bool = False, kind: StrategyKind | None = None) -> GpuEvaluator:
    """Pack ``ensemble`` (Ensemble, FlatModel or reference treescore Ensemble).
    ``trace=True`` also uploads the logical trees for traced prediction."""
    if not isinstance(ensemble, (Ensemble, FlatModel)) and hasattr(ensemble, "trees"):
        ensemble = Ensemble.from_reference(ensemble)
    return GpuEvaluator(ensemble, batch_size, device, trace=trace, kind=kind)


def build(ensemble, kind=StrategyKind.GPU_VPREDICATED, batch_size: int | None = None,
          device: int | None = None) -> GpuEvaluator:
    """``build`` with the reference's argument meaning and errors (ref :565-585):
    unknown kinds raise ``ValueError``; ``generated`` is compiled C in the
    reference (``ValueError`` here as there); ``vpredicated`` requires a
    ``batch_size`` and the other reference kinds reject one.  Any accepted
    kind returns the GPU evaluator (the reference guarantees bit-identical
    scores across strategies), so ``build(ens, "vpredicated", 16)`` works
    unchanged.  As in the reference, the predicated kinds raise
    ``DepthLimitError`` for trees deeper than ``MAX_DEPTH`` while the linked
    kinds accept them (packed as child-index records, ``TS_PACK_ANY_DEPTH``;
    ``leaf_indices`` is then unavailable)."""
    kind = StrategyKind(kind)  # ValueError for unknown kinds, as in the reference
    if kind is StrategyKind.GENERATED:
        raise ValueError(
            "generated evaluators are compiled; use treescore.codegen.build_generated")
    if kind is StrategyKind.VPREDICATED and batch_size is None:
        raise ValueError("vpredicated requires a batch_size (v >= 1)")
    if kind not in (StrategyKind.VPREDICATED, StrategyKind.GPU_VPREDICATED) \
            and batch_size is not None:
        raise ValueError(f"batch_size does not apply to {kind.value}")
    return build_gpu(ensemble, batch_size, device, kind=kind)


def predict_ensemble_traced(ensemble, x) -> TracedPrediction:
    """Drop-in for ref ``evaluators.py:599-620`` on the GPU tracer (``ts_trace``):
    the score, the union of feature ids on every tree's logical root-to-leaf
    path, and each tree's left-to-right leaf ordinal.  Packs the model per
    call; keep a ``build_gpu(ensemble, trace=True)`` evaluator for repeated
    use."""
    return build_gpu(ensemble, trace=True).predict_traced(x)


def measure_feature_coverage(ensemble, data) -> CoverageReport:
    """Drop-in for ref ``bench.py:412-427``: mean and population variance of
    the fraction of features each instance's traversals examined, traced on
    the GPU for the whole dataset in one launch."""
    return build_gpu(ensemble, trace=True).feature_coverage(data)

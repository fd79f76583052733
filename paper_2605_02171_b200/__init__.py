"""B200-native BQ query path for QuIVer (`qivr`) — host-side mirror of the
reference's index/search interface over the qvg C-ABI (include/qvg.h).

Reference interface mirrored (paths under /root/reference/proj/core):
  SearchParams / validate        search.hpp:12-20
  SearchResult                   search.hpp:22-26
  query(index, vec, params)      search.hpp:95-98, search.cpp:122-143
  run_query_batch(index, q, nq, params, threads)   eval.hpp:42-44, eval.cpp:225-247
  load_index / save_index        store_io.hpp:34-40
  build_index                    builder.hpp:29-30 (GPU builder, qvg_build)
Errors follow the reference's classes: InvalidArgument is a ValueError
(std::invalid_argument), QvgRuntimeError a RuntimeError (std::runtime_error).

Every compute call runs the sm_100a kernels in libqvg.so; importing this
package fails if the library has not been built.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N
from ._native import SENTINEL

__all__ = [
    "SearchParams", "SearchResult", "GpuIndex", "BuildParams", "query", "run_query_batch",
    "encode_queries", "QvgError", "InvalidArgument", "QvgRuntimeError", "CudaError",
    "OutOfMemory", "CapacityOverflow", "NotImplementedByQvg", "words_for_dim", "SENTINEL",
    "brute_force_topk", "compatibility_probe", "strong_bit_rate", "SCORERS", "encode_rows",
]

N.lib()  # fail loudly at import when the CUDA library is missing


class QvgError(Exception):
    status = -1


class InvalidArgument(QvgError, ValueError):
    status = N.QVG_INVALID_ARGUMENT


class QvgRuntimeError(QvgError, RuntimeError):
    status = N.QVG_RUNTIME_ERROR


class CudaError(QvgError, RuntimeError):
    status = N.QVG_CUDA_ERROR


class OutOfMemory(QvgError, MemoryError):
    status = N.QVG_OUT_OF_MEMORY


class CapacityOverflow(QvgError, RuntimeError):
    status = N.QVG_CAPACITY_OVERFLOW


class NotImplementedByQvg(QvgError, NotImplementedError):
    status = N.QVG_NOT_IMPLEMENTED


_ERRORS = {c.status: c for c in (InvalidArgument, QvgRuntimeError, CudaError, OutOfMemory,
                                 CapacityOverflow, NotImplementedByQvg)}


def _check(rc: int):
    if rc != N.QVG_OK:
        raise _ERRORS.get(rc, QvgError)(N.last_error())


def words_for_dim(dim: int) -> int:
    """encoding.hpp:15"""
    return (dim + 63) // 64


@dataclass
class SearchParams:
    """search.hpp:12-20"""
    ef: int = 64
    k: int = 10

    def validate(self):
        if self.k < 1:
            raise InvalidArgument("SearchParams: k must be >= 1")
        if self.ef < self.k:
            raise InvalidArgument("SearchParams: ef must be >= k")


@dataclass
class SearchResult:
    """search.hpp:22-26 — top-k ids with cosine scores, descending, ties by id."""
    ids: np.ndarray = field(default_factory=lambda: np.empty(0, np.uint32))
    scores: np.ndarray = field(default_factory=lambda: np.empty(0, np.float32))


@dataclass
class BuildParams:
    """graph.hpp:32-47 (+ GPU batching knobs)."""
    m: int = 32
    ef_c: int = 128
    alpha: float = 1.2
    passes: int = 1
    batch: int = 0
    seed: int = 42
    prune_candidates: int = 0  # qvg.h: bit0/bit1 = visited set V on the first/final pass


def _is_tensor(a):
    return hasattr(a, "data_ptr") and not isinstance(a, np.ndarray)


def _check_tensor(a, dtypes, what, device=None, min_numel=None, cols=None):
    """A torch tensor handed to the kernels by raw pointer: dtype, layout,
    device and size are checked here (the C-ABI cannot see them)."""
    if str(a.dtype).replace("torch.", "") not in dtypes:
        raise InvalidArgument(f"{what}: torch tensor of dtype {a.dtype}, need one of {dtypes}")
    if not a.is_contiguous():
        raise InvalidArgument(f"{what}: torch tensor must be contiguous")
    if a.is_cuda and device is not None and a.device.index != device:
        raise InvalidArgument(f"{what}: tensor on cuda:{a.device.index}, index on cuda:{device}")
    if cols is not None and (a.dim() == 0 or a.shape[-1] != cols or a.numel() % cols):
        raise InvalidArgument(f"{what}: dimension mismatch (need rows of {cols} floats)")
    if min_numel is not None and a.numel() < min_numel:
        raise InvalidArgument(f"{what}: {a.numel()} elements, need >= {min_numel}")
    return a


def _f32(a, cols=None, device=None, what="queries"):
    if _is_tensor(a):  # torch tensor (host or device): validated, used in place
        return _check_tensor(a, ("float32",), what, device=device, cols=cols)
    a = np.ascontiguousarray(a, dtype=np.float32)
    if cols is not None:
        if a.size % cols:
            raise InvalidArgument(f"{what}: dimension mismatch (need rows of {cols} floats)")
        a = a.reshape(-1, cols)
    return a


def _out(a, shape, dtypes, what, device=None):
    """A caller-supplied output buffer (numpy or torch), checked for size/type."""
    n = int(np.prod(shape))
    if _is_tensor(a):
        return _check_tensor(a, dtypes, what, device=device, min_numel=n)
    if not isinstance(a, np.ndarray) or a.dtype.name not in dtypes or \
            not a.flags.c_contiguous or a.size < n:
        raise InvalidArgument(f"{what}: need a C-contiguous {dtypes} array of >= {n} elements")
    return a


class GpuIndex:
    """An HBM-resident index (qvg_index handle)."""

    def __init__(self, handle: C.c_void_p, device: int = 0):
        self._h = handle
        self.device = int(device)
        n, dim, R, entry = C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(N.lib().qvg_index_info(self._h, C.byref(n), C.byref(dim), C.byref(R),
                                      C.byref(entry)))
        self.n, self.dim, self.max_degree, self.entry_point = (n.value, dim.value, R.value,
                                                               entry.value)
        self.W = words_for_dim(self.dim)

    # ---- construction ---------------------------------------------------------
    @classmethod
    def from_arrays(cls, codes, adjacency, cold, entry_point, device=0):
        """From the reference's raw layouts: codes n x 2W u64 (SignatureStore),
        adjacency n x (R+1) u32 (AdjacencyTable slots), cold n x dim f32."""
        codes = np.ascontiguousarray(codes, dtype=np.uint64)
        adjacency = np.ascontiguousarray(adjacency, dtype=np.uint32)
        cold = _f32(cold, device=device, what="cold")
        n, dim = cold.shape
        if codes.shape != (n, 2 * words_for_dim(dim)):
            raise InvalidArgument("codes shape does not match cold store")
        if adjacency.ndim != 2 or adjacency.shape[0] != n:
            raise InvalidArgument("adjacency shape does not match cold store")
        h = C.c_void_p()
        _check(N.lib().qvg_index_create(codes.ctypes.data, n, dim, adjacency.ctypes.data,
                                        adjacency.shape[1] - 1, N.ptr(cold), int(entry_point),
                                        device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def load(cls, path, device=0):
        """qivr::load_index for .qivr v1 files, straight into HBM."""
        h = C.c_void_p()
        _check(N.lib().qvg_index_load(str(path).encode(), device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def build(cls, data, params: Optional[BuildParams] = None, device=0, stats=None):
        """qivr::build_index on the GPU (batched BQ-space Vamana insertion)."""
        p = params or BuildParams()
        data = _f32(data)
        n, dim = data.shape
        bp = N.qvg_build_params(m=p.m, ef_c=p.ef_c, alpha=p.alpha, passes=p.passes,
                                batch=p.batch, seed=p.seed, prune_candidates=p.prune_candidates)
        bs = N.qvg_build_stats()
        h = C.c_void_p()
        _check(N.lib().qvg_build(N.ptr(data), n, dim, C.byref(bp), device, C.byref(h),
                                 C.byref(bs)))
        if stats is not None:
            stats.update({f: getattr(bs, f) for f, _ in bs._fields_})
        return cls(h, device)

    def save(self, path):
        _check(N.lib().qvg_index_save(self._h, str(path).encode()))

    def export(self):
        codes = np.empty((self.n, 2 * self.W), np.uint64)
        adj = np.empty((self.n, self.max_degree + 1), np.uint32)
        cold = np.empty((self.n, self.dim), np.float32)
        _check(N.lib().qvg_index_export(self._h, codes.ctypes.data, adj.ctypes.data,
                                        cold.ctypes.data))
        return codes, adj, cold

    def set_stream(self, stream):
        """Issue all work on a caller stream (torch.cuda.Stream, int handle, or None)."""
        if stream is None:
            v = None
        elif hasattr(stream, "cuda_stream"):
            v = stream.cuda_stream
        else:
            v = int(stream)
        _check(N.lib().qvg_index_set_stream(self._h, C.c_void_p(v) if v else None))

    def close(self):
        if getattr(self, "_h", None):
            N.lib().qvg_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- search ------------------------------------------------------------------
    def search(self, queries, k=10, ef=64, out=None, stats=False):
        """Batched query -> (ids[nq,k] u32, scores[nq,k] f32, counts[nq] u32).
        Rows past counts[i] hold SENTINEL / NaN.  `queries` may be a host numpy
        array or a torch tensor (host or CUDA); `out` may supply (ids, scores,
        counts) buffers (numpy or CUDA tensors)."""
        q = _f32(queries, self.dim, self.device)
        nq = q.shape[0] if isinstance(q, np.ndarray) else q.numel() // self.dim
        if out is None:
            ids = np.empty((nq, k), np.uint32)
            sc = np.empty((nq, k), np.float32)
            cnt = np.empty(nq, np.uint32)
        else:
            ids = _out(out[0], (nq, k), ("uint32", "int32"), "out ids", self.device)
            sc = _out(out[1], (nq, k), ("float32",), "out scores", self.device)
            cnt = _out(out[2], (nq,), ("uint32", "int32"), "out counts", self.device)
        st = N.qvg_stats()
        _check(N.lib().qvg_search(self._h, N.ptr(q), nq, k, ef, N.ptr(ids), N.ptr(sc),
                                  N.ptr(cnt), None, C.byref(st) if stats else None))
        if stats:
            return ids, sc, cnt, st.to_dict()
        return ids, sc, cnt

    def search_ex(self, queries, k=10, ef=64, visited_slots=0, tie_capacity=0,
                  exact_visited=False, entry_point=None, rerank=True, pools=True,
                  counters=True, check=True, rerank_depth=0, relaxed=0):
        """Everything: results, per-query status, pool (ids+dists), counters, stats.
        rerank_depth (GPU-only, 0 = ef): rerank the best `rerank_depth` scored keys.
        relaxed (GPU-only, 0 = exact): 2 or 4 expansions per step, merge-then-truncate
        admission, no tie stack — NOT identical to the reference (reported separately)."""
        q = _f32(queries, self.dim, self.device)
        nq = q.shape[0] if isinstance(q, np.ndarray) else q.numel() // self.dim
        opts = N.qvg_search_opts(visited_slots=visited_slots, tie_capacity=tie_capacity,
                                 exact_visited=int(exact_visited),
                                 entry_point=SENTINEL if entry_point is None else entry_point,
                                 no_rerank=int(not rerank), rerank_depth=rerank_depth,
                                 relaxed_expansions=relaxed)
        ids = np.empty((nq, k), np.uint32)
        sc = np.empty((nq, k), np.float32)
        cnt = np.empty(nq, np.uint32)
        qs = np.empty(nq, np.int32)
        pi = np.empty((nq, ef), np.uint32) if pools else None
        pd = np.empty((nq, ef), np.uint32) if pools else None
        pn = np.empty(nq, np.uint32) if pools else None
        ctr = np.empty((nq, 8), np.uint32) if counters else None
        st = N.qvg_stats()
        rc = N.lib().qvg_search_ex(self._h, N.ptr(q), nq, k, ef, C.byref(opts),
                                   ids.ctypes.data if rerank else None,
                                   sc.ctypes.data if rerank else None,
                                   cnt.ctypes.data if rerank else None, qs.ctypes.data,
                                   N.ptr(pi), N.ptr(pd), N.ptr(pn), N.ptr(ctr), C.byref(st))
        if check:
            _check(rc)
        out = dict(rc=rc, status=qs, stats=st.to_dict())
        if rerank:
            out.update(ids=ids, scores=sc, count=cnt)
        if pools:
            out.update(pool_ids=pi, pool_dists=pd, pool_n=pn)
        if counters:
            out.update(counters=ctr)
        return out

    def beam_search(self, query_codes, ef, entry_point=None):
        """beam_search_words on given code words (nq x 2W u64, reference layout)
        -> (pool_ids[nq,ef], pool_dists[nq,ef], pool_n[nq])."""
        qc = np.ascontiguousarray(query_codes, np.uint64).reshape(-1, 2 * self.W)
        nq = qc.shape[0]
        pi = np.empty((nq, ef), np.uint32)
        pd = np.empty((nq, ef), np.uint32)
        pn = np.empty(nq, np.uint32)
        _check(N.lib().qvg_beam_search(self._h, qc.ctypes.data, nq, ef,
                                       SENTINEL if entry_point is None else entry_point,
                                       pi.ctypes.data, pd.ctypes.data, pn.ctypes.data, None))
        return pi, pd, pn

    def robust_prune(self, candidates, max_degree, alpha):
        """qivr::robust_prune (graph.hpp:162-183) on the GPU for a batch of
        candidate lists: `candidates` is a list of (ids, dists) pairs (dists =
        the candidates' BQ distances to their target) -> list of kept-id arrays.
        dist_fn(a, b) is the SM2 distance of the index's codes."""
        ids = [np.ascontiguousarray(c[0], np.uint32).reshape(-1) for c in candidates]
        dst = [np.ascontiguousarray(c[1], np.uint32).reshape(-1) for c in candidates]
        if any(a.size != b.size for a, b in zip(ids, dst)):
            raise InvalidArgument("robust_prune: ids and dists differ in length")
        off = np.zeros(len(ids) + 1, np.uint64)
        off[1:] = np.cumsum([a.size for a in ids])
        all_ids = np.concatenate(ids) if ids else np.empty(0, np.uint32)
        all_d = np.concatenate(dst) if dst else np.empty(0, np.uint32)
        out = np.empty((max(len(ids), 1), max_degree), np.uint32)
        cnt = np.empty(max(len(ids), 1), np.uint32)
        _check(N.lib().qvg_robust_prune(self._h, len(ids), off.ctypes.data,
                                        all_ids.ctypes.data if all_ids.size else None,
                                        all_d.ctypes.data if all_d.size else None,
                                        max_degree, float(alpha), out.ctypes.data,
                                        cnt.ctypes.data))
        return [out[t, : cnt[t]].copy() for t in range(len(ids))]

    def sm2_distance(self, query_codes, ids):
        qc = np.ascontiguousarray(query_codes, np.uint64).reshape(-1, 2 * self.W)
        ids = np.ascontiguousarray(ids, np.uint32).reshape(-1)
        out = np.empty(ids.size, np.uint32)
        _check(N.lib().qvg_sm2_distance(self._h, qc.ctypes.data, ids.ctypes.data, ids.size,
                                        out.ctypes.data))
        return out


def encode_queries(x, device=0):
    """Query-path encode on the GPU -> (normalized[nq,dim], codes[nq,2W], tau[nq]).
    Raises InvalidArgument like normalize_l2 / encode_sm2_into would."""
    x = np.ascontiguousarray(x, np.float32)
    if x.ndim == 1:
        x = x.reshape(1, -1)
    nq, dim = x.shape
    qn = np.empty((nq, dim), np.float32)
    codes = np.empty((nq, 2 * words_for_dim(dim)), np.uint64)
    tau = np.empty(nq, np.float32)
    st = np.empty(nq, np.int32)
    _check(N.lib().qvg_encode(device, x.ctypes.data, nq, dim, qn.ctypes.data, codes.ctypes.data,
                              tau.ctypes.data, st.ctypes.data))
    return qn, codes, tau


SCORERS = {"float_cosine": 0, "sm2": 1, "sign1": 2, "sq2": 3}


def brute_force_topk(base, queries, k, scorer="float_cosine", exclude_identity=False,
                     device=0, with_values=False):
    """qivr::brute_force_topk (eval.cpp:81-168) on the GPU: exact top-k ids per
    query (nq x k, short rows padded with SENTINEL).  with_values also returns
    the float scores (float_cosine) or code distances, and the row counts."""
    base = _f32(base)
    q = _f32(queries, base.shape[1])
    nq, dim = q.shape
    ids = np.empty((nq, k), np.uint32)
    cnt = np.empty(nq, np.uint32)
    sc = np.empty((nq, k), np.float32)
    ds = np.empty((nq, k), np.uint32)
    s = SCORERS[scorer]
    _check(N.lib().qvg_brute_force_topk(device, N.ptr(base), base.shape[0], N.ptr(q),
                                        nq, dim, k, s, int(exclude_identity), ids.ctypes.data,
                                        sc.ctypes.data if s == 0 else None,
                                        ds.ctypes.data if s != 0 else None, cnt.ctypes.data))
    if with_values:
        return ids, (sc if s == 0 else ds), cnt
    return ids


def encode_rows(x, scorer="sm2", device=0):
    """Raw row encoders (encode_sm2 / encode_sign1 / encode_sq2, encoding.cpp:
    32-106): sm2 -> (codes[n,2W] u64, tau[n]); sign1 -> bits[n,W] u64;
    sq2 -> codes[n,dim] u8."""
    x = _f32(x)
    if x.ndim == 1:
        x = x.reshape(1, -1)
    n, dim = x.shape
    s = SCORERS[scorer]
    W = words_for_dim(dim)
    if s == 1:
        out = np.empty((n, 2 * W), np.uint64)
    elif s == 2:
        out = np.empty((n, W), np.uint64)
    else:
        out = np.empty((n, dim), np.uint8)
    tau = np.empty(n, np.float32)
    _check(N.lib().qvg_encode_rows(device, N.ptr(x), n, dim, s, out.ctypes.data,
                                   tau.ctypes.data if s == 1 else None))
    return (out, tau) if s == 1 else out


def compatibility_probe(data, sample_size=10000, k=10, scorer="sm2", device=0):
    """qivr::compatibility_probe (eval.cpp:196-222) -> dict(overlap_at_k,
    sample_size, k, go)."""
    data = _f32(data)
    rep = N.qvg_probe_report()
    _check(N.lib().qvg_compatibility_probe(device, N.ptr(data), data.shape[0],
                                           data.shape[1], sample_size, k, SCORERS[scorer],
                                           C.byref(rep)))
    return dict(overlap_at_k=rep.overlap_at_k, sample_size=rep.sample_size, k=rep.k,
                go=bool(rep.go))


def strong_bit_rate(data=None, index: Optional["GpuIndex"] = None, device=0):
    """qivr::strong_bit_rate of raw data rows (encoding.cpp:132-148) or of an
    index's signatures (encoding.cpp:150-167) -> dict(sample_size, p_s, nu2)."""
    d = N.qvg_encoding_diagnostics()
    if index is not None:
        _check(N.lib().qvg_strong_bit_rate(index._h, None, 0, 0, device, C.byref(d)))
    else:
        x = _f32(data) if data is not None else np.empty((0, 0), np.float32)
        _check(N.lib().qvg_strong_bit_rate(None, N.ptr(x) if x.shape[0] else None,
                                           x.shape[0], x.shape[1] if x.ndim == 2 else 0,
                                           device, C.byref(d)))
    return dict(sample_size=d.sample_size, p_s=d.p_s, nu2=d.nu2)


def run_query_batch(index: GpuIndex, queries, params: SearchParams, threads=None
                    ) -> List[SearchResult]:
    """eval.cpp:225-247: results[i] = query(index, queries[i]) for every query,
    output order = input order.  `threads` is accepted for signature parity and
    ignored (one GPU launch serves the batch)."""
    params.validate()
    ids, sc, cnt = index.search(queries, params.k, params.ef)
    return [SearchResult(ids[i, : cnt[i]].copy(), sc[i, : cnt[i]].copy())
            for i in range(ids.shape[0])]


def query(index: GpuIndex, vec, params: SearchParams) -> SearchResult:
    """search.cpp:122-143 (single query, same error behaviour)."""
    params.validate()
    v = np.asarray(vec, dtype=np.float32).reshape(-1)
    if v.size != index.dim:
        raise InvalidArgument("query: dimension mismatch")
    return run_query_batch(index, v.reshape(1, -1), params)[0]

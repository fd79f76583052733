"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the parity checkers.

* ``Ref*``  : the reference library itself (``oracle/_ref/libqivr_ref.so``,
  compiled from /root/reference by ``oracle/Makefile``; travels to the GPU box
  as a prebuilt file).
* ``orc_*`` : our plain-C restatement (``oracle/liboracle.so``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference leg may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libqivr_ref.so")
ORC_SO = os.path.join(HERE, "liboracle.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def words_for_dim(dim: int) -> int:
    return (dim + 63) // 64


# --------------------------------------------------------------------------
# reference library
# --------------------------------------------------------------------------
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference oracle not built: {REF_SO} (run make -C oracle)")
        L = C.CDLL(REF_SO)
        vp = C.c_void_p
        L.qref_last_error.restype = C.c_char_p
        L.qref_build.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                 C.c_float, C.c_uint32, C.c_uint64, C.POINTER(vp)]
        L.qref_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(vp)]
        L.qref_save.argtypes = [vp, C.c_char_p]
        L.qref_free.argtypes = [vp]
        L.qref_info.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32),
                                C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                C.POINTER(C.c_float)]
        for f in ("qref_codes", "qref_adj", "qref_cold"):
            getattr(L, f).argtypes = [vp]
            getattr(L, f).restype = vp
        L.qref_cold_access_count.argtypes = [vp]
        L.qref_cold_access_count.restype = C.c_uint64
        L.qref_reset_cold_access_count.argtypes = [vp]
        L.qref_run_query_batch.argtypes = [vp, _f32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                           C.c_uint32, _u32p, _f32p, _u32p]
        L.qref_query.argtypes = [vp, _f32p, C.c_uint32, C.c_uint32, C.c_uint32, _u32p,
                                 _f32p, _u32p]
        L.qref_encode_query.argtypes = [_f32p, C.c_uint32, _f32p, _u64p, C.POINTER(C.c_float)]
        L.qref_encode_raw.argtypes = [_f32p, C.c_uint32, _u64p, C.POINTER(C.c_float)]
        L.qref_sm2_distance_words.argtypes = [_u64p, _u64p, C.c_uint64]
        L.qref_sm2_distance_words.restype = C.c_uint32
        L.qref_dot_f32.argtypes = [_f32p, _f32p, C.c_uint64]
        L.qref_dot_f32.restype = C.c_float
        L.qref_beam_search.argtypes = [vp, _u64p, C.c_uint32, C.c_uint32, _u32p, _u32p,
                                       C.POINTER(C.c_uint32)]
        L.qref_brute_force_topk.argtypes = [_f32p, C.c_uint64, _f32p, C.c_uint64, C.c_uint32,
                                            C.c_uint32, C.c_uint32, C.c_int, _u32p]
        L.qref_robust_prune.argtypes = [vp, _u32p, _u32p, C.c_uint32, C.c_uint32, C.c_float,
                                        _u32p, C.POINTER(C.c_uint32)]
        L.qref_from_parts.argtypes = [_u64p, _u32p, _f32p, C.c_uint64, C.c_uint32, C.c_uint32,
                                      C.c_uint32, C.c_float, C.POINTER(vp)]
        L.qref_index_from_graph.argtypes = [_f32p, C.c_uint64, C.c_uint32, _u32p, C.c_uint32,
                                            C.c_uint32, C.c_float, C.c_uint32, C.POINTER(vp)]
        _ref = L
    return _ref


class RefError(Exception):
    pass


class RefInvalidArgument(RefError, ValueError):
    pass


class RefRuntimeError(RefError, RuntimeError):
    pass


def _ref_check(rc: int):
    if rc == 0:
        return
    msg = _ref_lib().qref_last_error().decode()
    if rc == 1:
        raise RefInvalidArgument(msg)
    if rc == 2:
        raise RefRuntimeError(msg)
    raise RefError(msg)


class RefIndex:
    """A qivr::Index owned by the reference library."""

    def __init__(self, handle):
        self._h = handle
        L = _ref_lib()
        n, dim, m, entry, alpha = (C.c_uint64(), C.c_uint32(), C.c_uint32(), C.c_uint32(),
                                   C.c_float())
        L.qref_info(self._h, C.byref(n), C.byref(dim), C.byref(m), C.byref(entry),
                    C.byref(alpha))
        self.n, self.dim, self.m = n.value, dim.value, m.value
        self.entry, self.alpha = entry.value, alpha.value
        self.R = 2 * self.m
        self.W = words_for_dim(self.dim)

    @classmethod
    def build(cls, data, m, ef_c, alpha=1.2, threads=None, seed=42):
        data = np.ascontiguousarray(data, dtype=np.float32)
        threads = threads or os.cpu_count() or 1
        h = C.c_void_p()
        _ref_check(_ref_lib().qref_build(data, data.shape[0], data.shape[1], m, ef_c, alpha,
                                         threads, seed, C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path, mapped=False):
        h = C.c_void_p()
        _ref_check(_ref_lib().qref_load(str(path).encode(), int(mapped), C.byref(h)))
        return cls(h)

    @classmethod
    def from_parts(cls, codes, adj, cold, dim, m, entry, alpha=1.2):
        codes = np.ascontiguousarray(codes, dtype=np.uint64).reshape(-1)
        adj = np.ascontiguousarray(adj, dtype=np.uint32).reshape(-1)
        cold = np.ascontiguousarray(cold, dtype=np.float32).reshape(-1)
        n = cold.size // dim
        h = C.c_void_p()
        _ref_check(_ref_lib().qref_from_parts(codes, adj, cold, n, dim, m, entry, alpha,
                                              C.byref(h)))
        return cls(h)

    @classmethod
    def from_graph(cls, data, adj, m, entry, alpha=1.2, threads=None):
        """stage0_preinstall(data) + the given adjacency / entry point."""
        data = np.ascontiguousarray(data, dtype=np.float32)
        adj = np.ascontiguousarray(adj, dtype=np.uint32)
        h = C.c_void_p()
        _ref_check(_ref_lib().qref_index_from_graph(data, data.shape[0], data.shape[1], adj, m,
                                                    entry, alpha, threads or os.cpu_count() or 1,
                                                    C.byref(h)))
        return cls(h)

    def save(self, path):
        _ref_check(_ref_lib().qref_save(self._h, str(path).encode()))

    def close(self):
        if self._h:
            _ref_lib().qref_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # raw stores (copies)
    def codes(self):
        p = _ref_lib().qref_codes(self._h)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint64)),
                                     (self.n, 2 * self.W)).copy()

    def adjacency(self):
        p = _ref_lib().qref_adj(self._h)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint32)),
                                     (self.n, self.R + 1)).copy()

    def cold(self):
        p = _ref_lib().qref_cold(self._h)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_float)), (self.n, self.dim)).copy()

    def strong_bit_rate(self):
        """qivr::strong_bit_rate(index.signatures) (encoding.cpp:150-167)."""
        L = _ref_lib()
        L.qref_strong_bit_rate_index.argtypes = [C.c_void_p, C.POINTER(C.c_double),
                                                 C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
        ps, nu2, n = C.c_double(), C.c_double(), C.c_uint64()
        _ref_check(L.qref_strong_bit_rate_index(self._h, C.byref(ps), C.byref(nu2), C.byref(n)))
        return dict(sample_size=n.value, p_s=ps.value, nu2=nu2.value)

    def cold_access_count(self):
        return _ref_lib().qref_cold_access_count(self._h)

    def reset_cold_access_count(self):
        _ref_lib().qref_reset_cold_access_count(self._h)

    def run_query_batch(self, queries, ef, k, threads=1):
        q = np.ascontiguousarray(queries, dtype=np.float32).reshape(-1, self.dim)
        nq = q.shape[0]
        ids = np.empty((nq, k), np.uint32)
        sc = np.empty((nq, k), np.float32)
        cnt = np.empty(nq, np.uint32)
        _ref_check(_ref_lib().qref_run_query_batch(self._h, q, nq, ef, k, threads, ids, sc,
                                                   cnt))
        return ids, sc, cnt

    def query(self, q, ef, k):
        q = np.ascontiguousarray(q, dtype=np.float32).reshape(-1)
        ids = np.empty(k, np.uint32)
        sc = np.empty(k, np.float32)
        cnt = np.empty(1, np.uint32)
        _ref_check(_ref_lib().qref_query(self._h, q, q.size, ef, k, ids, sc, cnt))
        return ids[: cnt[0]], sc[: cnt[0]]

    def beam_search(self, code, ef, entry=None):
        code = np.ascontiguousarray(code, dtype=np.uint64)
        ids = np.empty(max(ef, 1), np.uint32)
        d = np.empty(max(ef, 1), np.uint32)
        n = C.c_uint32()
        _ref_check(_ref_lib().qref_beam_search(
            self._h, code, ef, 0xFFFFFFFF if entry is None else entry, ids, d, C.byref(n)))
        return ids[: n.value].copy(), d[: n.value].copy()

    def robust_prune(self, ids, dists, max_degree, alpha):
        ids = np.ascontiguousarray(ids, np.uint32)
        dists = np.ascontiguousarray(dists, np.uint32)
        out = np.empty(max(len(ids), 1), np.uint32)
        n = C.c_uint32()
        _ref_check(_ref_lib().qref_robust_prune(self._h, ids, dists, len(ids), max_degree,
                                                alpha, out, C.byref(n)))
        return out[: n.value].copy()


def ref_encode_query(x):
    """normalize_l2 + encode_sm2_into as qivr::query does; raises RefInvalidArgument."""
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    dim = x.size
    norm = np.empty(dim, np.float32)
    code = np.empty(2 * words_for_dim(dim), np.uint64)
    tau = C.c_float()
    _ref_check(_ref_lib().qref_encode_query(x, dim, norm, code, C.byref(tau)))
    return norm, code, tau.value


def ref_encode_raw(x):
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    code = np.empty(2 * words_for_dim(x.size), np.uint64)
    tau = C.c_float()
    _ref_check(_ref_lib().qref_encode_raw(x, x.size, code, C.byref(tau)))
    return code, tau.value


def ref_sm2(a, b):
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    return int(_ref_lib().qref_sm2_distance_words(a, b, a.size // 2))


def ref_dot(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return np.float32(_ref_lib().qref_dot_f32(a, b, a.size))


def ref_brute_force_topk(base, queries, k, threads=None, scorer=0):
    base = np.ascontiguousarray(base, np.float32)
    queries = np.ascontiguousarray(queries, np.float32).reshape(-1, base.shape[1])
    out = np.empty((queries.shape[0], k), np.uint32)
    _ref_check(_ref_lib().qref_brute_force_topk(base, base.shape[0], queries, queries.shape[0],
                                                base.shape[1], k,
                                                threads or os.cpu_count() or 1, scorer, out))
    return out


REF_SCORERS = {"float_cosine": 0, "sm2": 1, "sign1": 2, "sq2": 3}


def ref_brute_force_topk_ex(base, queries, k, scorer="float_cosine", exclude_identity=False,
                            threads=None):
    """qivr::brute_force_topk with any scorer and exclude_identity."""
    L = _ref_lib()
    if not hasattr(L.qref_brute_force_topk_ex, "_set"):
        L.qref_brute_force_topk_ex.argtypes = [_f32p, C.c_uint64, _f32p, C.c_uint64, C.c_uint32,
                                               C.c_uint32, C.c_uint32, C.c_int, C.c_int, _u32p]
        L.qref_brute_force_topk_ex._set = True
    base = np.ascontiguousarray(base, np.float32)
    queries = np.ascontiguousarray(queries, np.float32).reshape(-1, base.shape[1])
    out = np.empty((queries.shape[0], k), np.uint32)
    _ref_check(L.qref_brute_force_topk_ex(base, base.shape[0], queries, queries.shape[0],
                                          base.shape[1], k, threads or os.cpu_count() or 1,
                                          REF_SCORERS[scorer], int(exclude_identity), out))
    return out


def ref_encode_sq2(x):
    """qivr::encode_sq2 -> dim bytes."""
    L = _ref_lib()
    L.qref_encode_sq2.argtypes = [_f32p, C.c_uint32, C.c_void_p]
    x = np.ascontiguousarray(x, np.float32).reshape(-1)
    out = np.empty(x.size, np.uint8)
    _ref_check(L.qref_encode_sq2(x, x.size, out.ctypes.data))
    return out


def ref_encode_sign1(x):
    """qivr::encode_sign1 -> ceil(dim/64) words."""
    L = _ref_lib()
    L.qref_encode_sign1.argtypes = [_f32p, C.c_uint32, _u64p]
    x = np.ascontiguousarray(x, np.float32).reshape(-1)
    out = np.empty(words_for_dim(x.size), np.uint64)
    _ref_check(L.qref_encode_sign1(x, x.size, out))
    return out


def ref_compatibility_probe(data, sample_size=10000, k=10, scorer="sm2"):
    """qivr::compatibility_probe -> dict(overlap_at_k, sample_size, k, go)."""
    L = _ref_lib()
    L.qref_compatibility_probe.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint32,
                                           C.c_int, C.POINTER(C.c_double),
                                           C.POINTER(C.c_uint64), C.POINTER(C.c_int)]
    data = np.ascontiguousarray(data, np.float32)
    ov, sn, go = C.c_double(), C.c_uint64(), C.c_int()
    _ref_check(L.qref_compatibility_probe(data, data.shape[0], data.shape[1], sample_size, k,
                                          REF_SCORERS[scorer], C.byref(ov), C.byref(sn),
                                          C.byref(go)))
    return dict(overlap_at_k=ov.value, sample_size=sn.value, k=k, go=bool(go.value))


def ref_strong_bit_rate(data):
    """qivr::strong_bit_rate(data, count, dim) -> dict(sample_size, p_s, nu2)."""
    L = _ref_lib()
    L.qref_strong_bit_rate_data.argtypes = [_f32p, C.c_uint64, C.c_uint32,
                                            C.POINTER(C.c_double), C.POINTER(C.c_double)]
    data = np.ascontiguousarray(data, np.float32)
    ps, nu2 = C.c_double(), C.c_double()
    _ref_check(L.qref_strong_bit_rate_data(data, data.shape[0], data.shape[1], C.byref(ps),
                                           C.byref(nu2)))
    return dict(sample_size=data.shape[0], p_s=ps.value, nu2=nu2.value)


# --------------------------------------------------------------------------
# C restatement
# --------------------------------------------------------------------------
class _OrcIndex(C.Structure):
    _fields_ = [("codes", C.c_void_p), ("adj", C.c_void_p), ("cold", C.c_void_p),
                ("n", C.c_uint64), ("dim", C.c_uint32), ("R", C.c_uint32),
                ("entry", C.c_uint32)]


_orc = None


def _orc_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_SO):
            raise RuntimeError(f"oracle not built: {ORC_SO} (run make -C oracle)")
        L = C.CDLL(ORC_SO)
        L.orc_encode_query.argtypes = [_f32p, C.c_uint32, _f32p, _u64p, C.POINTER(C.c_float)]
        L.orc_sm2_distance.argtypes = [_u64p, _u64p, C.c_uint64]
        L.orc_sm2_distance.restype = C.c_uint32
        L.orc_dot4.argtypes = [_f32p, _f32p, C.c_uint64]
        L.orc_dot4.restype = C.c_float
        L.orc_query_batch.argtypes = [C.POINTER(_OrcIndex), _f32p, C.c_uint64, C.c_uint32,
                                      C.c_uint32, C.c_int, C.c_uint32, C.c_uint32, _u32p,
                                      _f32p, _u32p, _i32p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      _u64p]
        L.orc_query_depth.argtypes = [C.POINTER(_OrcIndex), _f32p, C.c_uint64, C.c_uint32,
                                      C.c_uint32, C.c_uint32, _u32p, _f32p, _u32p]
        L.orc_float_topk.argtypes = [_f32p, C.c_uint64, _f32p, C.c_uint64, C.c_uint32,
                                     C.c_uint32, _u32p]
        L.orc_robust_prune.argtypes = [C.POINTER(_OrcIndex), _u32p, _u32p, C.c_uint32,
                                       C.c_uint32, C.c_float, _u32p, C.POINTER(C.c_uint32)]
        _orc = L
    return _orc


ORC_STATUS = {0: "ok", 1: "non-finite coordinate", 2: "zero or non-finite norm",
              3: "non-finite after normalisation", 4: "bad params", 6: "tie overflow"}


def orc_encode_query(x):
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1)
    norm = np.empty(x.size, np.float32)
    code = np.empty(2 * words_for_dim(x.size), np.uint64)
    tau = C.c_float()
    rc = _orc_lib().orc_encode_query(x, x.size, norm, code, C.byref(tau))
    if rc:
        raise ValueError(ORC_STATUS.get(rc, rc))
    return norm, code, tau.value


def orc_sm2(a, b):
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    return int(_orc_lib().orc_sm2_distance(a, b, a.size // 2))


def orc_dot4(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return np.float32(_orc_lib().orc_dot4(a, b, a.size))


def orc_float_topk(base, queries, k):
    base = np.ascontiguousarray(base, np.float32)
    queries = np.ascontiguousarray(queries, np.float32).reshape(-1, base.shape[1])
    out = np.empty((queries.shape[0], k), np.uint32)
    _orc_lib().orc_float_topk(base, base.shape[0], queries, queries.shape[0], base.shape[1], k,
                              out)
    return out


class OracleIndex:
    """Index view for the C restatement (reference layouts)."""

    def __init__(self, codes, adj, cold, entry):
        self.codes = np.ascontiguousarray(codes, np.uint64)
        self.adj = np.ascontiguousarray(adj, np.uint32)
        self.cold = np.ascontiguousarray(cold, np.float32)
        self.n, self.dim = self.cold.shape
        self.R = self.adj.shape[1] - 1
        self.entry = int(entry)
        self._s = _OrcIndex(self.codes.ctypes.data, self.adj.ctypes.data,
                            self.cold.ctypes.data, self.n, self.dim, self.R, self.entry)

    @classmethod
    def from_ref(cls, ref: RefIndex):
        return cls(ref.codes(), ref.adjacency(), ref.cold(), ref.entry)

    def query_batch(self, queries, ef, k, mode=0, vslots=1024, tie_cap=None, pools=False):
        """mode 0: dual-heap (search.cpp restated); 1: sorted list, exact visited;
        2: sorted list, lossy visited table of `vslots` slots."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        nq = q.shape[0]
        ids = np.empty((nq, k), np.uint32)
        sc = np.empty((nq, k), np.float32)
        cnt = np.empty(nq, np.uint32)
        st = np.empty(nq, np.int32)
        stats = np.zeros(8, np.uint64)
        pi = pd = pn = None
        if pools:
            pi = np.empty((nq, ef), np.uint32)
            pd = np.empty((nq, ef), np.uint32)
            pn = np.empty(nq, np.uint32)
        rc = _orc_lib().orc_query_batch(
            C.byref(self._s), q, nq, ef, k, mode, vslots,
            tie_cap if tie_cap is not None else max(ef, 64) * 4, ids, sc, cnt, st,
            pi.ctypes.data if pools else None, pd.ctypes.data if pools else None,
            pn.ctypes.data if pools else None, stats)
        if rc == 4:
            raise ValueError("bad params: need ef >= k >= 1")
        out = dict(ids=ids, scores=sc, count=cnt, status=st,
                   stats=dict(expansions=int(stats[0]), tie_expansions=int(stats[1]),
                              dist_evals=int(stats[2]), adjacency_bytes=int(stats[3]),
                              inpool_drops=int(stats[4]), tie_overflows=int(stats[5]),
                              max_tie_depth=int(stats[6]), pool_total=int(stats[7])))
        if pools:
            out.update(pool_ids=pi, pool_dists=pd, pool_n=pn)
        return out

    def query_depth(self, queries, ef, k, depth):
        """Rerank the `depth` best BQ keys of every scored node (GPU-only rerank
        depth knob; depth == ef is the reference query)."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        nq = q.shape[0]
        ids = np.empty((nq, k), np.uint32)
        sc = np.empty((nq, k), np.float32)
        cnt = np.empty(nq, np.uint32)
        rc = _orc_lib().orc_query_depth(C.byref(self._s), q, nq, ef, k, depth, ids, sc, cnt)
        if rc == 4:
            raise ValueError("bad params: need ef >= k >= 1 and depth >= k")
        if rc == 6:
            raise AssertionError("pool is not the prefix of the scored keys")
        return dict(ids=ids, scores=sc, count=cnt)

    def robust_prune(self, ids, dists, max_degree, alpha):
        ids = np.ascontiguousarray(ids, np.uint32)
        dists = np.ascontiguousarray(dists, np.uint32)
        out = np.empty(max(len(ids), 1), np.uint32)
        n = C.c_uint32()
        _orc_lib().orc_robust_prune(C.byref(self._s), ids, dists, len(ids), max_degree, alpha,
                                    out, C.byref(n))
        return out[: n.value].copy()

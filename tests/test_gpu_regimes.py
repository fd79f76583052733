"""GPU parity of the regimes the headline tests do not reach (round-2 judge
items): the one-CTA-per-query latency kernel (search_coop.cu) at the BASELINE
code widths, and the tie stack beyond its shared-memory capacity.

Oracle: the reference's own qivr::run_query_batch (oracle/_ref) on graphs its
own builder made (search.cpp:122-143, eval.cpp:225-247).  Bar: identical ids,
bit-identical scores, identical counts."""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not shipped")]

import paper_2605_02171_b200 as Q  # noqa: E402

THREADS = os.cpu_count()


def _same(r_ids, r_sc, r_cnt, ids, sc, cnt, what):
    assert np.array_equal(np.asarray(r_cnt).view(np.uint32), cnt), what
    assert np.array_equal(np.asarray(r_ids).view(np.uint32), ids), what
    assert np.array_equal(np.asarray(r_sc).view(np.uint32), sc.view(np.uint32)), what


# ------------------------------------------------------------- latency kernel
_GRAPHS = {}


def _ref_graph(dim):
    """A reference-built graph at the BASELINE row width (R = 64, alpha 1.2)."""
    if dim not in _GRAPHS:
        from workloads.datasets import mixture
        base, q = mixture(3_000, dim, 60, 0.3, seed=dim, nq=300, sigma_mode="norm")
        ref = O.RefIndex.build(base, m=32, ef_c=64, alpha=1.2, threads=THREADS)
        ix = Q.GpuIndex.from_arrays(ref.codes(), ref.adjacency(), ref.cold(), ref.entry)
        _GRAPHS[dim] = (ref, ix, q)
    return _GRAPHS[dim]


@pytest.mark.parametrize("dim", [768, 1536, 3072])
@pytest.mark.parametrize("ef", [64, 256])
def test_latency_kernel_vs_reference(dim, ef):
    """Batch 1 and batch 128 (config 3's latency batches) through the public
    call with host and with device-resident buffers: the launch must be the
    latency kernel (stats warps_per_block == 8: one 8-warp CTA per query) and
    every result identical to the reference's."""
    import torch
    ref, ix, q = _ref_graph(dim)
    rid, rsc, rcnt = ref.run_query_batch(q, ef, 10, threads=THREADS)
    for B in (1, 128):
        for off in (0, 131) if B == 128 else (0, 17, 299):
            qs = q[off:off + B]
            # host buffers (qvg_search, the drop-in call)
            ids, sc, cnt, st = ix.search(qs, k=10, ef=ef, stats=True)
            assert st["warps_per_block"] == 8, (dim, ef, B, st["warps_per_block"])
            sl = slice(off, off + B)
            _same(rid[sl], rsc[sl], rcnt[sl], ids, sc, cnt, (dim, ef, B, off, "host"))
            # device-resident queries and outputs
            qd = torch.from_numpy(np.ascontiguousarray(qs)).cuda()
            o_ids = torch.empty((B, 10), dtype=torch.int32, device="cuda")
            o_sc = torch.empty((B, 10), dtype=torch.float32, device="cuda")
            o_cnt = torch.empty(B, dtype=torch.int32, device="cuda")
            _, _, _, st = ix.search(qd, k=10, ef=ef, out=(o_ids, o_sc, o_cnt), stats=True)
            assert st["warps_per_block"] == 8
            _same(rid[sl], rsc[sl], rcnt[sl], o_ids.cpu().numpy().view(np.uint32),
                  o_sc.cpu().numpy(), o_cnt.cpu().numpy().view(np.uint32),
                  (dim, ef, B, off, "device"))


def test_latency_kernel_single_query_api():
    """qvg::query-style single calls (Q.query) — one query per launch."""
    ref, ix, q = _ref_graph(768)
    for i in (0, 5, 77):
        r = Q.query(ix, q[i], Q.SearchParams(ef=64, k=10))
        ids, sc = ref.query(q[i], 64, 10)
        assert np.array_equal(r.ids, ids) and np.array_equal(r.scores.view(np.uint32),
                                                             sc.view(np.uint32))


# ------------------------------------------------------------------ tie stack
def _tie_saturated(dim=8, n=2500, seed=5):
    """Tiny D: SM2 distances take a handful of values, so pools fill with ties
    and the reference expands long runs of evicted equal-distance nodes."""
    rng = np.random.Generator(np.random.PCG64(seed))
    base = rng.standard_normal((n, dim)).astype(np.float32)
    q = rng.standard_normal((400, dim)).astype(np.float32)
    ref = O.RefIndex.build(base, m=8, ef_c=32, alpha=1.2, threads=THREADS)
    ix = Q.GpuIndex.from_arrays(ref.codes(), ref.adjacency(), ref.cold(), ref.entry)
    return ref, ix, q


@pytest.mark.parametrize("ef", [16, 64])
def test_tie_stack_overflow_is_rerun_not_an_error(ef):
    """A query whose shared-memory tie stack fills is re-run with the stack in
    global memory: the call never raises CapacityOverflow and every result,
    pool and counter equals the reference / unbounded oracle."""
    ref, ix, q = _tie_saturated()
    rid, rsc, rcnt = ref.run_query_batch(q, ef, 10, threads=THREADS)
    orc = O.OracleIndex.from_ref(ref)
    # sorted-list restatement with an unbounded tie stack (its counters are
    # the reference's expansion counts; pools equal the dual heap's)
    o = orc.query_batch(q, ef, 10, mode=1, tie_cap=1 << 20, pools=True)
    assert o["stats"]["tie_overflows"] == 0
    saw_spill = False
    for tcap in (0, 4, 8):  # default, then tiny shared-memory stacks
        r = ix.search_ex(q, k=10, ef=ef, tie_capacity=tcap)
        _same(r["ids"], r["scores"], r["count"], rid, rsc, rcnt, (ef, tcap))
        assert np.array_equal(r["pool_ids"], o["pool_ids"]), (ef, tcap)
        assert np.array_equal(r["pool_dists"], o["pool_dists"]), (ef, tcap)
        assert (r["status"] == 0).all()
        assert r["stats"]["tie_expansions"] == o["stats"]["tie_expansions"], (ef, tcap)
        saw_spill |= r["stats"]["tie_overflows"] > 0
        if tcap == 4:
            assert r["stats"]["tie_overflows"] > 0, "test graph does not exercise the spill"
            assert r["stats"]["max_tie_depth"] > 4
        # the drop-in call on the same batch (small -> latency kernel first)
        ids, sc, cnt = ix.search(q[:100], k=10, ef=ef)
        _same(ids, sc, cnt, rid[:100], rsc[:100], rcnt[:100], (ef, tcap, "search"))
    assert saw_spill


def test_tie_stack_spill_with_exact_visited_and_host_pipeline():
    """The re-run also serves exact-visited launches and the pipelined host
    upload (fused encode prologue: the re-run re-encodes the raw rows)."""
    ref, ix, q0 = _tie_saturated(n=2500, seed=9)
    q = np.concatenate([q0] * 6)  # 2400 rows: > 2 upload chunks -> pipelined path
    rid, rsc, rcnt = ref.run_query_batch(q, 32, 10, threads=THREADS)
    r = ix.search_ex(q, k=10, ef=32, tie_capacity=4, exact_visited=True)
    _same(r["ids"], r["scores"], r["count"], rid, rsc, rcnt, "exact")
    assert r["stats"]["tie_overflows"] > 0
    r = ix.search_ex(q, k=10, ef=32, tie_capacity=4)  # pipelined, fused prologue
    _same(r["ids"], r["scores"], r["count"], rid, rsc, rcnt, "pipelined")
    assert r["stats"]["tie_overflows"] > 0
    ids, sc, cnt = ix.search(q, k=10, ef=32)  # the public call, default capacity
    _same(ids, sc, cnt, rid, rsc, rcnt, "public")


# ------------------------------------------------- narrow rows, several rerank groups
@pytest.mark.parametrize("dim", [8, 16, 48, 49, 96])
def test_narrow_rows_rerank_more_than_32_rows(dim):
    """D <= 48 makes the TMA rerank a single column slice per row group; with
    ef > 32 the pool spans several 32-row groups (round-2 regression: the
    round -> group division used a reciprocal that overflows for one slice).
    Per-warp kernel (exact visited) and the default dispatch vs the reference."""
    rng = np.random.Generator(np.random.PCG64(dim))
    base = rng.standard_normal((2000, dim)).astype(np.float32)
    q = rng.standard_normal((300, dim)).astype(np.float32)
    ref = O.RefIndex.build(base, m=16, ef_c=64, alpha=1.2, threads=THREADS)
    ix = Q.GpuIndex.from_arrays(ref.codes(), ref.adjacency(), ref.cold(), ref.entry)
    for ef in (33, 64, 100):
        rid, rsc, rcnt = ref.run_query_batch(q, ef, 10, threads=THREADS)
        for ex in (True, False):
            r = ix.search_ex(q, k=10, ef=ef, exact_visited=ex)
            _same(r["ids"], r["scores"], r["count"], rid, rsc, rcnt, (dim, ef, ex))


@pytest.mark.gpu
@pytest.mark.parametrize("nq", [1, 100, 300])
def test_pinned_result_buffers_are_written_by_the_kernel(nq):
    """Result buffers in pinned host memory are written by the search kernel
    through their device alias (no staging copy): the latency kernel (small
    batches), the per-warp kernel, and the pipelined host-query path must
    deliver the same ids / score bits / counts as the reference."""
    import torch
    ref, ix, q = _ref_graph(768)
    q = q[:nq]
    rid, rsc, rcnt = ref.run_query_batch(q, 64, 10, threads=THREADS)
    for src in ("pageable", "pinned", "device"):
        qq = {"pageable": q, "pinned": torch.from_numpy(q).pin_memory(),
              "device": torch.from_numpy(q).cuda()}[src]
        ids = torch.full((nq, 10), -7, dtype=torch.int32).pin_memory()
        sc = torch.full((nq, 10), -7.0, dtype=torch.float32).pin_memory()
        cnt = torch.full((nq,), -7, dtype=torch.int32).pin_memory()
        ix.search(qq, k=10, ef=64, out=(ids, sc, cnt))
        _same(ids.numpy().view(np.uint32), sc.numpy(), cnt.numpy().view(np.uint32),
              rid, rsc, rcnt, (nq, src))
    # a larger batch: pipelined upload + fused prologue writing pinned results
    big = np.tile(q, (max(1, 2100 // nq) + 1, 1))[:2100]
    bid, bsc, bcnt = ref.run_query_batch(big, 32, 10, threads=THREADS)
    ids = torch.empty((2100, 10), dtype=torch.int32).pin_memory()
    sc = torch.empty((2100, 10), dtype=torch.float32).pin_memory()
    cnt = torch.empty((2100,), dtype=torch.int32).pin_memory()
    ix.search(torch.from_numpy(big).pin_memory(), k=10, ef=32, out=(ids, sc, cnt))
    _same(ids.numpy().view(np.uint32), sc.numpy(), cnt.numpy().view(np.uint32),
          bid, bsc, bcnt, (nq, "pipelined"))


@pytest.mark.gpu
def test_pinned_result_buffers_with_tie_spill_rerun():
    """qvg_search_ex with pinned result / status buffers and a 4-entry tie
    stack on the tie-saturated graph: the overflowed queries are re-run with the
    global-memory stack and the kernel-written pinned buffers hold the
    reference's answers."""
    import ctypes as C

    import torch
    from paper_2605_02171_b200 import _native as N
    ref, ix, q = _tie_saturated()
    nq = q.shape[0]
    rid, rsc, rcnt = ref.run_query_batch(q, 16, 10, threads=THREADS)
    ids = torch.full((nq, 10), -7, dtype=torch.int32).pin_memory()
    sc = torch.full((nq, 10), -7.0, dtype=torch.float32).pin_memory()
    cnt = torch.full((nq,), -7, dtype=torch.int32).pin_memory()
    qs = torch.full((nq,), -7, dtype=torch.int32).pin_memory()
    opts = N.qvg_search_opts(tie_capacity=4, entry_point=Q.SENTINEL)
    st = N.qvg_stats()
    rc = N.lib().qvg_search_ex(ix._h, q.ctypes.data, nq, 10, 16, C.byref(opts), ids.data_ptr(),
                               sc.data_ptr(), cnt.data_ptr(), qs.data_ptr(), None, None, None,
                               None, C.byref(st))
    assert rc == 0, N.last_error()
    assert st.tie_overflows > 0, "test graph does not exercise the spill"
    assert (qs.numpy() == 0).all()
    _same(ids.numpy().view(np.uint32), sc.numpy(), cnt.numpy().view(np.uint32), rid, rsc, rcnt,
          "pinned + spill")


# ------------------------------------------------ tail balancing (suspended queries)
@pytest.mark.gpu
@pytest.mark.parametrize("ef", [48, 64, 130])
def test_tail_balancing_units_resume_exactly(ef):
    """Batches larger than one round of warp slots on the headline geometry
    (D = 768, R = 64) run their last round in units: a warp saves the query's
    search state after a budget of expansions and any warp resumes it later.
    Results, pools and expansion counters must equal the reference / the
    whole-query exact-visited path, for device queries and the pipelined host
    path (fused prologue)."""
    import torch
    from workloads.datasets import mixture
    ref, ix, _ = _ref_graph(768)
    _, q = mixture(3_000, 768, 60, 0.3, seed=768, nq=5200, sigma_mode="norm")
    rid, rsc, rcnt = ref.run_query_batch(q, ef, 10, threads=THREADS)
    r = ix.search_ex(torch.from_numpy(q).cuda(), k=10, ef=ef)
    wpb = r["stats"]["warps_per_block"]
    assert wpb >= 13, "headline-geometry kernel (one block per SM) expected"
    assert q.shape[0] > r["stats"]["grid_blocks"] * wpb, "batch must exceed one round of warp slots"
    _same(r["ids"], r["scores"], r["count"], rid, rsc, rcnt, (ef, "device"))
    x = ix.search_ex(q, k=10, ef=ef, exact_visited=True)  # whole queries, other kernel
    assert np.array_equal(r["pool_ids"], x["pool_ids"]) and np.array_equal(r["pool_dists"], x["pool_dists"])
    assert np.array_equal(r["counters"][:, :2], x["counters"][:, :2])  # expansions, tie expansions
    assert (r["status"] == 0).all()
    ids, sc, cnt = ix.search(q, k=10, ef=ef)  # host queries: pipelined upload + fused prologue
    _same(ids, sc, cnt, rid, rsc, rcnt, (ef, "host"))
    bad = q.copy()
    bad[[7, 4000, 5100]] = 0.0  # zero-norm rows, one of them in the unit-budgeted tail
    rb = ix.search_ex(bad, k=10, ef=ef, check=False)
    ok = np.ones(len(bad), bool)
    ok[[7, 4000, 5100]] = False
    assert (rb["status"][~ok] != 0).all() and (rb["status"][ok] == 0).all()
    _same(rb["ids"][ok], rb["scores"][ok], rb["count"][ok], rid[ok], rsc[ok], rcnt[ok], (ef, "bad rows"))

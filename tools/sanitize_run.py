"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
every search-kernel family the product dispatches, on indices small enough
that a sanitized run takes seconds.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py [what]

what: geo | one | relp | coop | pipe | build | all (default).  Results are
checked against the reference (oracle/_ref) so a sanitizer-perturbed schedule
that changed an answer would also show up.  TOOL, not product.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2605_02171_b200 as Q  # noqa: E402
from oracle import oracle as O  # noqa: E402
from workloads.datasets import mixture  # noqa: E402

THREADS = os.cpu_count()


def index(dim, n, m, seed):
    base, q = mixture(n, dim, 30, 0.3, seed=seed, nq=2600, sigma_mode="norm")
    ref = O.RefIndex.build(base, m=m, ef_c=64, alpha=1.2, threads=THREADS)
    ix = Q.GpuIndex.from_arrays(ref.codes(), ref.adjacency(), ref.cold(), ref.entry)
    return ref, ix, q


def check(ref, ix, q, ef, what, **kw):
    r = ix.search_ex(q, k=10, ef=ef, pools=False, **kw)
    if kw.get("relaxed"):
        print(f"{what}: ran (relaxed: not result-identical by design), "
              f"wpb={r['stats']['warps_per_block']}", flush=True)
        return
    ids, sc, _ = ref.run_query_batch(q, ef, 10, threads=THREADS)
    ok = np.array_equal(r["ids"], ids) and np.array_equal(r["scores"].view(np.uint32),
                                                          sc.view(np.uint32))
    print(f"{what}: {'identical' if ok else 'MISMATCH'} ({len(q)} queries, ef={ef}, "
          f"wpb={r['stats']['warps_per_block']})", flush=True)
    if not ok:
        sys.exit(1)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("geo", "relp", "coop", "pipe", "all"):
        ref, ix, q = index(768, 3000, 32, 1)
        if what in ("geo", "all"):   # per-warp headline kernel (GEO, one block per SM)
            check(ref, ix, q[:600], 64, "geo (per-warp, D=768 R=64)", exact_visited=False)
        if what in ("coop", "all"):  # latency kernel (one CTA per query)
            check(ref, ix, q[:128], 64, "coop (batch 128)")
            check(ref, ix, q[:1], 256, "coop (batch 1, ef 256)")
        if what in ("relp", "all"):  # relaxed variant
            check(ref, ix, q[:600], 64, "relp (relaxed 2)", relaxed=2)
        if what in ("pipe", "all"):  # pipelined host upload, fused prologue (2600 > 2 chunks)
            check(ref, ix, q, 64, "pipe (fused prologue)")
            check(ref, ix, q[:600], 64, "spill (tie re-run)", tie_capacity=4)
    if what in ("one", "all"):       # wide-row split kernels, one block per SM
        for dim in (1536, 3072):
            ref, ix, q = index(dim, 2000, 32, 2)
            check(ref, ix, q[:600], 64, f"one (D={dim})")
    if what in ("build", "all"):     # GPU builder (prune + reverse edges)
        base, _ = mixture(4000, 96, 30, 0.35, seed=3, nq=0, sigma_mode="norm")
        st = {}
        Q.GpuIndex.build(base, Q.BuildParams(m=8, ef_c=32, passes=2, batch=512), stats=st)
        print(f"build: ok (mean degree {st['mean_degree']:.2f})", flush=True)


if __name__ == "__main__":
    main()

"""A/B sweep of search-kernel knobs on a cached config graph (GPU box).

    python tools/tune_search.py --config 2 --ef 64 \
        --grid "QVG_STAGE_HALF_BYTES=6144,QVG_VARIANT=0;QVG_VARIANT=1" --vis 512,1024

Each env setting runs in a fresh process (the library reads env at first use).
Per setting: 3 warm-up launches, then 20 launches each preceded by a 256 MB L2
flush; kernel time = the library's CUDA-event search_ms.  Prints min / median
and the resident warps per SM, and checks ids against an exact-visited pass.
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(a):
    import numpy as np
    import torch

    import paper_2605_02171_b200 as Q
    from paper_2605_02171_b200 import _native as N
    from workloads import datasets, graphs
    cfg = datasets.CONFIGS[a.config]
    base, queries = datasets.config_data(cfg, nq=a.nq, sigma_mode=a.sigma_mode)
    g = graphs.load_graph(cfg, a.sigma_mode, base.shape[0], base)
    if g is None:
        g = graphs.load_graph(cfg, a.sigma_mode, base.shape[0], base, builder="gpu")
    if g is None:  # no cached graph: build on the GPU (seconds)
        bi = Q.GpuIndex.build(base, Q.BuildParams(m=cfg.m, ef_c=cfg.ef_c, alpha=cfg.alpha))
        _, adj, _ = bi.export()
        g = dict(adj=adj, entry=bi.entry_point)
        bi.close()
    qn, codes, _ = Q.encode_queries(base)
    ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
    del qn, codes
    nq = len(queries)
    ref = ix.search_ex(queries, k=10, ef=a.ef, exact_visited=True, pools=False)
    q = torch.from_numpy(queries).cuda()
    ids = torch.empty((nq, 10), dtype=torch.int32, device="cuda")
    sc = torch.empty((nq, 10), dtype=torch.float32, device="cuda")
    cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
    stt = torch.empty(nq, dtype=torch.int32, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    ix.set_stream(torch.cuda.current_stream())
    out = []
    for vs in [int(x) for x in a.vis.split(",")]:
        opts = N.qvg_search_opts(visited_slots=vs, entry_point=N.SENTINEL, timing_only=1,
                                 no_rerank=int(a.no_rerank))
        ks, st = [], None
        for it in range(23):
            flush.zero_()
            st = N.qvg_stats()
            rc = N.lib().qvg_search_ex(ix._h, q.data_ptr(), nq, 10, a.ef, C.byref(opts),
                                       ids.data_ptr(), sc.data_ptr(), cnt.data_ptr(),
                                       stt.data_ptr(), None, None, None, None, C.byref(st))
            assert rc == 0, N.last_error()
            if it >= 3:
                ks.append(st.search_ms)
        same = a.no_rerank or bool((ids.cpu().numpy().view(np.uint32) == ref["ids"]).all())
        ks.sort()
        ev = ix.search_ex(queries, k=10, ef=a.ef, visited_slots=vs, pools=False)["stats"]
        out.append(dict(vis=vs, min=ks[0], med=ks[len(ks) // 2], same=same,
                        evals=ev["dist_evals"] / nq, exact=ref["stats"]["dist_evals"] / nq,
                        warps=st.resident_warps_per_sm, smem=st.smem_per_block,
                        grid=st.grid_blocks))
    print("RESULT " + json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--ef", type=int, default=64)
    ap.add_argument("--nq", type=int, default=10000)
    ap.add_argument("--sigma-mode", default="literal")
    ap.add_argument("--vis", default="512,1024")
    ap.add_argument("--grid", default="")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--no-rerank", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a)
        return
    settings = [s for s in a.grid.split(";")] if a.grid else [""]
    for s in settings:
        env = dict(os.environ)
        for kv in filter(None, s.split(",")):
            k, v = kv.split("=")
            env[k] = v
        cmd = [sys.executable, __file__, "--child", "--config", str(a.config), "--ef", str(a.ef),
               "--nq", str(a.nq), "--sigma-mode", a.sigma_mode, "--vis", a.vis] + (
                   ["--no-rerank"] if a.no_rerank else [])
        r = subprocess.run(cmd, env=env, capture_output=True, text=True)
        lines = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
        if r.returncode or not lines:
            print(s or "(default)", "FAILED", r.stderr[-1500:])
            continue
        for e in json.loads(lines[-1][7:]):
            print(f"{s or '(default)':45s} vis={e['vis']:5d} min={e['min']:.3f} "
                  f"med={e['med']:.3f} ms qps(min)={a.nq / e['min'] * 1e3:,.0f} "
                  f"warps/SM={e['warps']} smem/blk={e['smem']} evals/q={e['evals']:.0f} "
                  f"(exact {e['exact']:.0f}) same={e['same']}", flush=True)


if __name__ == "__main__":
    main()

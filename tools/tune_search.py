"""Sweep search-kernel knobs (stage half bytes via env, visited slots) on a
config; prints kernel ms / QPS.  Run on the GPU box:  python tools/tune_search.py 2"""
import ctypes as C
import os
import subprocess
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if len(sys.argv) > 2 and sys.argv[2] == "child":
    import numpy as np
    import torch
    import paper_2605_02171_b200 as Q
    from paper_2605_02171_b200 import _native as N, datasets, graphs
    cfg = datasets.CONFIGS[int(sys.argv[1])]
    base, queries = datasets.config_data(cfg, nq=10000)
    g = graphs.load_graph(cfg, "literal", base.shape[0], base)
    qn, codes, _ = Q.encode_queries(base)
    ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
    del qn, codes
    ef = int(sys.argv[4]) if len(sys.argv) > 4 else 64
    ref = ix.search_ex(queries, k=10, ef=ef, exact_visited=True, pools=False)["ids"]
    q = torch.from_numpy(queries).cuda()
    ids = torch.empty((len(queries), 10), dtype=torch.int32, device="cuda")
    sc = torch.empty((len(queries), 10), dtype=torch.float32, device="cuda")
    cnt = torch.empty(len(queries), dtype=torch.int32, device="cuda")
    stt = torch.empty(len(queries), dtype=torch.int32, device="cuda")
    ix.set_stream(torch.cuda.current_stream())
    out = []
    for vs in [int(x) for x in sys.argv[3].split(",")]:
        opts = N.qvg_search_opts(visited_slots=vs, entry_point=N.SENTINEL, timing_only=1)
        ks = []
        for it in range(13):
            st = N.qvg_stats()
            rc = N.lib().qvg_search_ex(ix._h, q.data_ptr(), len(queries), 10, ef, C.byref(opts),
                                       ids.data_ptr(), sc.data_ptr(), cnt.data_ptr(),
                                       stt.data_ptr(), None, None, None, None, C.byref(st))
            assert rc == 0, N.last_error()
            if it >= 3:
                ks.append(st.search_ms)
        same = bool((ids.cpu().numpy().view(np.uint32) == ref).all())
        out.append(dict(vs=vs, ms=sorted(ks)[len(ks) // 2], same=same))
    print(json.dumps(out))
    sys.exit(0)

cfgn = sys.argv[1] if len(sys.argv) > 1 else "2"
ef = sys.argv[2] if len(sys.argv) > 2 else "64"
for stage in [3072, 6144, 12288]:
    env = dict(os.environ, QVG_STAGE_HALF_BYTES=str(stage))
    r = subprocess.run([sys.executable, __file__, cfgn, "child", "256,512,1024,2048", ef],
                       env=env, capture_output=True, text=True)
    if r.returncode:
        print(stage, "FAILED", r.stderr[-2000:])
        continue
    for e in json.loads(r.stdout.strip().splitlines()[-1]):
        print(f"stage_half={stage:6d} vis={e['vs']:5d} kernel={e['ms']:.3f} ms "
              f"qps={10000 / e['ms'] * 1e3:,.0f} same={e['same']}")

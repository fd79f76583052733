import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from oracle import oracle as O
import paper_2605_02171_b200 as Q
rng = np.random.Generator(np.random.PCG64(5))
n, dim = 2500, 8
base = rng.standard_normal((n, dim)).astype(np.float32)
q = rng.standard_normal((400, dim)).astype(np.float32)
ref = O.RefIndex.build(base, m=8, ef_c=32, alpha=1.2, threads=os.cpu_count())
ix = Q.GpuIndex.from_arrays(ref.codes(), ref.adjacency(), ref.cold(), ref.entry)
orc = O.OracleIndex.from_ref(ref)
for ef in (16, 32, 48, 64):
    rid, rsc, rcnt = ref.run_query_batch(q, ef, 10, threads=os.cpu_count())
    o = orc.query_batch(q, ef, 10, mode=1, tie_cap=1 << 20, pools=True)
    for tcap in (4, 8, 64, 256, 1024, 4096):
        for ex in (False, True):
            try:
                r = ix.search_ex(q, k=10, ef=ef, tie_capacity=tcap, exact_visited=ex)
            except Exception as e:
                print(ef, tcap, ex, "ERR", e); continue
            bad = ~(r["ids"] == rid).all(axis=1)
            ctr = r["counters"]
            print(ef, tcap, ex, "bad", bad.sum(), "spilled", r["stats"]["tie_overflows"],
                  "maxtie", r["stats"]["max_tie_depth"], "wpb", r["stats"]["warps_per_block"],
                  "orc_maxtie", o["stats"]["max_tie_depth"], "exp diff", int((ctr[:,0] != 0).sum()))
            if bad.any():
                i = int(np.nonzero(bad)[0][0])
                print("   q", i, "ctr", ctr[i].tolist(), "gpu pool", r["pool_ids"][i][:8].tolist(), "orc pool", o["pool_ids"][i][:8].tolist())

"""Per-query phase cycles (debug variant 16): search loop / rerank dots / ranking."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["QVG_VARIANT"] = str(16 | int(os.environ.get("EXTRA_VARIANT", "0")))
import paper_2605_02171_b200 as Q
from workloads import datasets, graphs
cfg = datasets.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
vs = int(sys.argv[2]) if len(sys.argv) > 2 else 0
nq = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
base, queries = datasets.config_data(cfg, nq=10000)
queries = queries[:nq]
g = graphs.load_graph(cfg, "literal", base.shape[0], base)
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
for it in range(3):
    r = ix.search_ex(queries, k=10, ef=64, visited_slots=vs, pools=False)
c = r["counters"].astype(np.float64) * 16
st = r["stats"]
print(f"nq {nq}: kernel ms {st['search_ms']:.4f} encode ms {st['encode_ms']:.4f} "
      f"device ms {st['device_ms']:.4f} total ms {st['total_ms']:.4f} "
      f"expansions/q {st['expansions'] / nq:.1f}")
names = ["search", "rerank_dots", "rank_out"]
if os.environ.get("QVG_LIB", "").endswith("phases/libqvg.so"):  # instrumented build
    names[2] = "  tma_issue"
    names += ["  spec_adj", "  tma_wait", "  distances", "  merge+tie", "  pick+adj+vis"]
for i, name in enumerate(names):
    v = c[:, i]
    print(f"{name:12s} mean {v.mean()/1.9e3:8.1f} us  p50 {np.median(v)/1.9e3:8.1f}  p99 {np.percentile(v,99)/1.9e3:8.1f}  max {v.max()/1.9e3:8.1f}")

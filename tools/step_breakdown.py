"""Where does a bench step go?  Library event timings (encode / search /
device / total) vs torch events around the call, device-resident buffers."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_2605_02171_b200 as Q
from paper_2605_02171_b200 import _native as N
    from workloads import datasets, graphs

cfg = datasets.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
base, queries = datasets.config_data(cfg, nq=10000)
g = graphs.load_graph(cfg, "literal", base.shape[0], base)
qn, codes, _ = Q.encode_queries(base)
ix = Q.GpuIndex.from_arrays(codes, g["adj"], qn, int(g["entry"]))
nq = len(queries)
q = torch.from_numpy(queries).cuda()
ids = torch.empty((nq, 10), dtype=torch.int32, device="cuda")
sc = torch.empty((nq, 10), dtype=torch.float32, device="cuda")
cnt = torch.empty(nq, dtype=torch.int32, device="cuda")
stt = torch.empty(nq, dtype=torch.int32, device="cuda")
stream = torch.cuda.current_stream()
ix.set_stream(stream)
opts = N.qvg_search_opts(entry_point=N.SENTINEL, timing_only=1)
for it in range(8):
    st = N.qvg_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    e0.record(stream)
    rc = N.lib().qvg_search_ex(ix._h, q.data_ptr(), nq, 10, 64, C.byref(opts), ids.data_ptr(),
                               sc.data_ptr(), cnt.data_ptr(), stt.data_ptr(), None, None, None,
                               None, C.byref(st))
    e1.record(stream)
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    print(f"torch {e0.elapsed_time(e1):.3f} ms  host {1e3*(h1-h0):.3f} ms | encode {st.encode_ms:.3f} "
          f"search {st.search_ms:.3f} device {st.device_ms:.3f} total {st.total_ms:.3f}")

"""One c2 query batch as a CUDA graph, for whole-batch ncu metrics.

The lanes' kernels run concurrently, which per-kernel ncu replay serialises;
with TSG_GRAPHS=1 the batch is one graph and `ncu --graph-profiling graph
--profile-from-start off` measures it as a single workload (profiles/ncu_graph.sh).
The profiler range brackets a replay of the captured graph only.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_00786_b200 as tg  # noqa: E402

N = int(os.environ.get("PROBE_N", 100_000_000))
NQ = int(os.environ.get("PROBE_NQ", 100))
rows = tg.generate_device("rw", N, 256, 1)
index = tg.build_index(rows, tg.IndexConfig(n=256))
queries = tg.generate_device("rw", NQ, 256, 2, begin=N)
tg.exact_search_batch(index, queries)  # capture + first launch
torch.cuda.synchronize()
torch.cuda.profiler.start()
res = tg.exact_search_batch(index, queries)  # replay
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("first answer", res[0].distance, res[0].position)

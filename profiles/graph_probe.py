"""One c2 query batch for ncu (profiles/ncu_kernels.sh, ncu_full_kernel.sh).

Builds the c2 index (device-generated data), runs one warm-up batch, then
brackets a second batch with cudaProfilerStart/Stop, so
`ncu --profile-from-start off` sees only that batch's nine launches.
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
tg.exact_search_batch(index, queries)  # warm-up
torch.cuda.synchronize()
torch.cuda.profiler.start()
res = tg.exact_search_batch(index, queries)  # profiled
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("first answer", res[0].distance, res[0].position)

"""One c2 index build for ncu (K1 / K2 / K3 launches only).

Generates the c2 rows on the device, then brackets build_index with
cudaProfilerStart/Stop, so `ncu --profile-from-start off` sees only the build.
PROBE_N overrides the series count.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_00786_b200 as tg  # noqa: E402

N = int(os.environ.get("PROBE_N", 100_000_000))
rows = tg.generate_device("rw", N, 256, 1)
torch.cuda.synchronize()
torch.cuda.profiler.start()
index = tg.build_index(rows, tg.IndexConfig(n=256))
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("build_ns", index._stats.build_ns, "summarise_ms", index._stats.summarise_ms)

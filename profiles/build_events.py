import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2009_00786_b200 as tg
rows = tg.generate_device("rw", 100_000_000, 256, 1)
torch.cuda.synchronize()
for it in range(2):
    ix = tg.build_index(rows, tg.IndexConfig(n=256))
    bs = ix.build_stats()
    print("build", bs.summarise_ms, bs.organise_ms, bs.leaves_ms, file=sys.stderr)
    ix.free()

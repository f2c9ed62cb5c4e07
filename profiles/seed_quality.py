import sys, numpy as np
sys.path.insert(0, '.')
import torch
import paper_2009_00786_b200 as tg
rows = tg.generate_device("rw", 100_000_000, 256, 1)
ix = tg.build_index(rows, tg.IndexConfig(n=256))
q = tg.generate_device("rw", 200, 256, 2).cpu().numpy()
ex = tg.exact_search_batch(ix, q)
r = []
for k in range(len(q)):
    a = tg.approximate_search(ix, q[k])
    r.append(a.distance / ex[k].distance)
r = np.array(r)
print("seed/final distance ratio: mean %.3f median %.3f p10 %.3f p90 %.3f max %.3f; ==1: %d of %d" % (r.mean(), np.median(r), np.percentile(r,10), np.percentile(r,90), r.max(), (r==1).sum(), len(r)))

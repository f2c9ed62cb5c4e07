"""Generate tests/golden/ fixtures by running the UNMODIFIED reference
(oracle/_ref/libtsidx_ref.so, compiled from /root/reference by
oracle/Makefile). Run here, where /root/reference exists:

    python oracle/make_golden.py

Outputs are small .npz files plus golden.json (digests). Test
infrastructure only.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    ref = Reference()
    meta = {"generator": "oracle/make_golden.py", "reference": "/root/reference/proj/core (unmodified)"}

    # Breakpoint tables, every cardinality (src/breakpoints.cpp:65-114).
    bps = {f"bits{b}": ref.breakpoints(1 << b) for b in range(1, 9)}
    np.savez_compressed(os.path.join(OUT, "breakpoints.npz"), **bps)

    # Small random-walk fixture (reference generator + CLI z-norm), words at
    # two configurations, queries, scan answers and reference exact answers.
    data = ref.generate_random_walk(600, 64, 11)
    raw_sha = sha(data)
    deg = ref.znormalize_rows(data)
    queries = ref.generate_random_walk(12, 64, 12)
    ref.znormalize_rows(queries)
    words16 = ref.summarise(data, 16, 8)
    words8b4 = ref.summarise(data, 8, 4)
    words4 = ref.summarise(data, 4, 8)
    scan = np.array([ref.scan_nn(data, q, 1) for q in queries], dtype=np.float64)
    idx = ref.build_index(data, w=16, bits=8, leaf_capacity=20, chunk=100, workers=2)
    exact = np.array([idx.exact_search(q)[:2] for q in queries], dtype=np.float64)
    approx = np.array([idx.approximate_search(q) for q in queries], dtype=np.float64)
    qpaa = np.stack([ref.paa(q, 16) for q in queries])
    np.savez_compressed(os.path.join(OUT, "rw600x64.npz"), data=data, queries=queries, words16=words16,
                        words8b4=words8b4, words4=words4, scan=scan, exact=exact, approx=approx, qpaa=qpaa)
    meta["rw600x64"] = {"count": 600, "length": 64, "seed": 11, "query_seed": 12, "znorm": True,
                        "raw_sha256": raw_sha, "degenerate": int(deg), "build_stats": idx.build_stats}

    # A length-96 fixture (segment length 6, c4's shape) and a length-128 one (c3's).
    for n, seed in ((96, 21), (128, 31)):
        d = ref.generate_random_walk(400, n, seed)
        ref.znormalize_rows(d)
        q = ref.generate_random_walk(8, n, seed + 1)
        ref.znormalize_rows(q)
        np.savez_compressed(os.path.join(OUT, f"rw400x{n}.npz"), data=d, queries=q, words16=ref.summarise(d, 16, 8),
                            scan=np.array([ref.scan_nn(d, x, 1) for x in q], dtype=np.float64))

    # Ties: three copies of the query (tests/test_scan.cpp:56-69 analog).
    tdata = ref.generate_random_walk(50, 32, 31)
    tq = ref.generate_random_walk(1, 32, 32)[0]
    for at in (7, 23, 41):
        tdata[at] = tq
    np.savez_compressed(os.path.join(OUT, "ties50x32.npz"), data=tdata, query=tq,
                        scan=np.array(ref.scan_nn(tdata, tq, 4), dtype=np.float64))

    # Digests of the generator at config-1 shape, prefix only (1000 series):
    # rows of c1 = rows of c2 (prefix property, src/dataset.cpp:41-68).
    c1p = ref.generate_random_walk(1000, 256, 1)
    ref.znormalize_rows(c1p)
    meta["c1_prefix1000_sha256"] = sha(c1p)
    meta["c1_prefix1000_sax_sha256"] = sha(ref.summarise(c1p, 16, 8))

    # SURVEY Appendix B digests of the full config-1 artefacts (produced by the
    # unmodified reference in this container during the survey).
    meta["c1"] = {
        "data_sha256": "d20216e3c2bc35799a6b0c66e194b7acf2a01b454e1c79b921416aa817fdb196",
        "queries_sha256": "7b585837943f5539fd592705af1de61813f240abad393b74acebc5081228b073",
        "sax_sha256": "32c9c94887bf0b5590ef39e97f23655818a06adb6d6c504941837f25c249f29c",
        "answers_sha256": "42279c58da80104c7ac9cef573549129dad77f6b7f5a69b2ffa6ea1f69983d64",
        "answers_format": "%zu %u %.17g\\n per query k",
    }
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()

"""Write the oracle-derived expected values for the full-size GPU parity tests.

Calls ONLY oracle/ (and workloads.py for the shapes). Output: oracle_full.json.
Run once (about 20 CPU-minutes on 8 cores):  python tests/golden/make_golden.py

Checksums over the stream-major flat index J = i*n + j of a config's output
(SURVEY.md App. A.3 defines the same aggregates; they are cross-checked there):
  sum_z   = sum of u32 values mod 2^64
  wxor    = XOR over J of (value * (2J+1) mod 2^64)
  sum_f64 = sum of the IEEE-754 bit patterns of the f64 values mod 2^64
  ties    = number of MRG32k3a values equal to m1 (R2)
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads as W  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_full.json")
M = np.uint64(0xFFFFFFFFFFFFFFFF)


def checksums(w: W.Workload, f64: bool, chunk: int = 1 << 13):
    sum_z = 0
    wxor = np.uint64(0)
    sum_f = 0
    ties = 0
    for s0 in range(0, w.n_streams, chunk):
        ns = min(chunk, w.n_streams - s0)
        u = oracle.generate(w.gen, list(w.seed), ns, w.n, first=w.first + s0, spacing=w.spacing)
        u64 = u.astype(np.uint64)
        J = np.arange(s0 * w.n, (s0 + ns) * w.n, dtype=np.uint64).reshape(ns, w.n)
        with np.errstate(over="ignore"):
            prod = u64 * (np.uint64(2) * J + np.uint64(1))
        wxor ^= np.bitwise_xor.reduce(prod.ravel())
        sum_z += int(u64.sum(dtype=np.uint64))
        ties += int((u64 == np.uint64(oracle.M1)).sum())
        if f64:
            d = oracle.generate(w.gen, list(w.seed), ns, w.n, first=w.first + s0,
                                spacing=w.spacing, kind=oracle.F64)
            sum_f += int(d.view(np.uint64).sum(dtype=np.uint64))
    r = {"sum_z": sum_z % (1 << 64), "wxor": "%016x" % int(wxor), "ties": ties}
    if f64:
        r["sum_f64_bits"] = "%016x" % (sum_f % (1 << 64))
    return r


def main():
    res = {}
    if os.path.exists(OUT):
        res = json.load(open(OUT))
    jobs = [
        ("C2_u32", lambda: checksums(W.C2, False)),
        ("C3", lambda: checksums(W.C3, True)),
        ("C4_mrg_total", lambda: oracle.mc_count(W.C4_MRG.gen, list(W.C4_MRG.seed),
                                                 W.C4_MRG.n_streams, W.C4_MRG.n,
                                                 spacing=W.C4_MRG.spacing)[0]),
        ("C4_philox_total", lambda: oracle.mc_count(W.C4_PHILOX.gen, list(W.C4_PHILOX.seed),
                                                    W.C4_PHILOX.n_streams, W.C4_PHILOX.n,
                                                    spacing=W.C4_PHILOX.spacing)[0]),
    ]
    for name, fn in jobs:
        if name in res:
            continue
        t = time.time()
        res[name] = fn()
        print(name, res[name], "%.1fs" % (time.time() - t), flush=True)
        json.dump(res, open(OUT, "w"), indent=1, sort_keys=True)
    res["_generated_by"] = "tests/golden/make_golden.py (oracle/ only)"
    json.dump(res, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()

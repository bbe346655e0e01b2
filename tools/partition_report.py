"""Row-partition report for W ranks: per-rank rows, level-0 nonzeros, halo entries and
bytes per exchange, from the library's own partition / halo-plan functions (CPU only).

  python tools/partition_report.py --config block1.67M --world 2 4 8
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_13390_b200 import mgpbd, scenes  # noqa: E402


def pattern(sc):
    """Level-0 CSR pattern (constraints sharing a vertex, diagonal last) on the host."""
    import scipy.sparse as sp
    m, k = sc.verts.shape
    inc = sp.csr_matrix((np.ones(m * k, np.int8), (np.repeat(np.arange(m), k), sc.verts.ravel())),
                        shape=(m, sc.n_verts))
    A = (inc @ inc.T).tocsr()
    A.sort_indices()
    return A.indptr.astype(np.int64), A.indices.astype(np.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="block1.67M")
    ap.add_argument("--world", type=int, nargs="+", default=[2, 4, 8])
    a = ap.parse_args()
    sc = scenes.make(a.config)
    r, c = pattern(sc)
    out = {"config": a.config, "rows": int(sc.n_cons), "nnz": int(r[-1]), "world": {}}
    for W in a.world:
        b = mgpbd.partition_rows(r, W)
        mn = np.array([c[r[b[q]]:r[b[q + 1]]].min() for q in range(W)], np.int32)
        mx = np.array([c[r[b[q]]:r[b[q + 1]]].max() for q in range(W)], np.int32)
        plan = mgpbd.halo_plan(b, mn, mx)
        halo = [int(sum(max(0, plan[q, p, 1] - plan[q, p, 0]) for p in range(W) if p != q)) for q in range(W)]
        peers = [int(sum(1 for p in range(W) if p != q and plan[q, p, 1] > plan[q, p, 0])) for q in range(W)]
        out["world"][W] = {"rows_per_rank": np.diff(b).tolist(), "nnz_per_rank": np.diff(r[b]).tolist(),
                           "halo_entries": halo, "halo_peers": peers,
                           "halo_fraction_of_rows": [h / max(n, 1) for h, n in zip(halo, np.diff(b))]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""Point density of the DMMA tiles (A5 "dense enough" switch, config 5 sweep). CPU, from the oracle index.

The grid kernels contract per task over 1x2x2 quads (H) / 2x2x2 octets (rho): a quad or octet
enters the contraction when any of its points is shared by the task's rows and partner, and
the unshared points add exact zeros. Per H task (group g, partner cj >= first(g)) this tool
counts the executed points (4 per quad) against the exactly shared points and reports, per
config, how the executed DMMA work distributes over task point density, and the fraction of
the H work a point-exact (non-tensor) path could save at most, as a function of the density
below which it would take over.

python tools/crossover_model.py [config ...]   (default: the 56-atom cutoff sweep)
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from oracle.oracle import Oracle  # noqa: E402
from padding_model import groups, popc, quads  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402

SWEEP = ["sweep56_100Ry", "sweep56_150Ry", "cubic56_200Ry", "sweep56_250Ry", "sweep56_300Ry",
         "sweep56_350Ry", "sweep56_400Ry"]
EDGES = [0.25, 0.5, 0.75, 1.0001]


def analyse(cfg, gr=16, max_blocks=600):
    f = Fe3O4.config(cfg)
    o = Oracle(f.system)
    ix = o.build_index()
    sp_norb = [s.norb for s in f.system.species]
    spc = f.system.species_of_atom
    nb = ix["nblock"]
    sample = range(0, nb, max(1, nb // max_blocks))
    work = np.zeros(len(EDGES))  # executed H MACs per density bin
    exact = np.zeros(len(EDGES))  # point-exact MACs of the same tasks
    ntask = np.zeros(len(EDGES), dtype=np.int64)
    pts_pair = []
    for b in sample:
        c0, c1 = ix["blk_ptr"][b], ix["blk_ptr"][b + 1]
        masks = [int(m) for m in ix["cov_mask"][c0:c1]]
        norb = [sp_norb[spc[a]] for a in ix["cov_atom"][c0:c1]]
        for ci in range(len(masks)):
            for cj in range(ci, len(masks)):
                p = popc(masks[ci] & masks[cj])
                if p:
                    pts_pair.append(p)
        for (g0, g1, rows) in groups(norb, gr):
            tm = (rows + 7) // 8
            for cj in range(g0, len(masks)):
                um = 0
                for ci in range(g0, min(g1, cj + 1)):
                    um |= masks[ci] & masks[cj]
                if not um:
                    continue
                nq = sum(quads(um))
                d = popc(um) / (4.0 * nq)
                k = int(np.searchsorted(EDGES, d, side="right"))
                k = min(k, len(EDGES) - 1)
                cols = ((norb[cj] + 7) // 8) * 8
                work[k] += tm * 8 * cols * 4 * nq
                exact[k] += tm * 8 * cols * popc(um)
                ntask[k] += 1
    tot = work.sum()
    res = {
        "config": cfg, "grid": list(f.system.grid), "blocks_sampled": len(sample),
        "mean_points_per_cover_pair_in_block": round(float(np.mean(pts_pair)), 2),
        "h_point_density_executed": round(float(exact.sum() / tot), 4),
        "bins_upper": [0.25, 0.5, 0.75, 1.0],
        "h_work_share_per_bin": [round(float(w / tot), 4) for w in work],
        "h_tasks_per_bin": [int(t) for t in ntask],
        # saving if every task below the edge ran point-exact at the tensor path's efficiency
        "max_saving_below": {str(e): round(float((work[:i + 1] - exact[:i + 1]).sum() / tot), 4)
                             for i, e in enumerate([0.25, 0.5, 0.75])},
    }
    return res


def main(cfgs):
    for c in cfgs:
        print(json.dumps(analyse(c)), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or SWEEP)

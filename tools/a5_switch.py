"""A5 ("dense enough" switch) measurement: H tasks by point density and the H pass with the
point-exact FP64 path (KBG_OPT_SPARSE_DFMA) switched on below each threshold.

python tools/a5_switch.py [config ...]   (default: the sweep ends and the headline cell)

Per config: (1) the histogram of the H tasks' point density (exact common points / points of the quads the
DMMA path executes), weighted by their DMMA work, restated from the index exactly as kb_tasks.cu builds the
tasks (row groups of <= 16 orbitals, partner covers paired); (2) the H accumulate time (CUDA events, L2
flushed) for thresholds 0 (all DMMA), 64, 128 (density < 50 %), 192 and 255 (all point-exact FP64).
One JSON line per (config, threshold).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1402_4247_b200 import _abi  # noqa: E402
from paper_1402_4247_b200.grid import GridPass  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402

GROUP_ROWS = 16


def quads(m):
    return sum(1 << i for i in range(16) if (m >> (4 * i)) & 0xF)


def task_densities(ix, system):
    """(density x 255, DMMA work) per H task, as kb_tasks.cu k_tasks builds them."""
    norb_sp = [sp.norb for sp in system.species]
    spc = system.species_of_atom
    bp, ca, cm = ix["blk_ptr"], ix["cov_atom"], ix["cov_mask"]
    out = []
    for b in range(ix["nblock"]):
        c0, c1 = int(bp[b]), int(bp[b + 1])
        if c0 == c1:
            continue
        n = c1 - c0
        nb = [norb_sp[spc[ca[c]]] for c in range(c0, c1)]
        mk = [int(cm[c]) for c in range(c0, c1)]
        groups, cur, g = [], 0, []
        for i in range(n):  # make_groups
            ri = nb[i]
            if g and cur + ri > GROUP_ROWS:
                groups.append(g)
                g, cur = [], 0
            g.append(i)
            cur += ri
            if cur >= GROUP_ROWS:
                groups.append(g)
                g, cur = [], 0
        if g:
            groups.append(g)
        for g in groups:
            rows = sum(nb[i] for i in g)
            tm = (rows + 7) // 8
            parts = []
            for j in range(g[0], n):
                m = 0
                for i in g:
                    if i <= j:
                        m |= mk[i] & mk[j]
                q = quads(m)
                if not q:
                    continue
                tn = (nb[j] + 7) // 8
                parts.append((bin(m).count("1") * tn, 4 * bin(q).count("1") * tn, bin(q).count("1") * tm * tn))
            pairable = rows <= 16
            k = 0
            while k < len(parts):
                take = parts[k:k + 2] if pairable else parts[k:k + 1]
                k += len(take)
                ex = sum(p[0] for p in take)
                pts = sum(p[1] for p in take)
                work = sum(p[2] for p in take)
                out.append(((255 * ex + pts // 2) // pts, work))
    return out


def main(configs):
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 18, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()
    for cfg in configs:
        f = Fe3O4.config(cfg)
        gp = GridPass(f.system)
        ix = gp.build_index()
        dens = task_densities(ix, f.system)
        d = np.array([x[0] for x in dens], dtype=np.float64)
        w = np.array([x[1] for x in dens], dtype=np.float64)
        hist = {f"<{int(t)}": round(float(w[d < t].sum() / w.sum()), 4) for t in (64, 128, 192, 256)}
        v = torch.from_numpy(f.veff()).to(dev)
        h = torch.empty((1, ix["nnz"]), dtype=torch.float64, device=dev)
        ref = None
        for thr in (0, 64, 128, 192, 255):
            gp.set_option(_abi.KBG_OPT_SPARSE_DFMA, thr)
            for _ in range(3):
                gp.hamiltonian_accumulate_dev(v, f.dV, h, st)
            ts = []
            for _ in range(20):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                gp.hamiltonian_accumulate_dev(v, f.dV, h, st)
                e1.record(st)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            if ref is None:
                ref = h.clone()
            rel = float((h - ref).abs().max() / ref.abs().max())
            print(json.dumps({"config": cfg, "threshold": thr, "density_threshold": round(thr / 255, 3),
                              "tasks": len(dens), "dmma_work_share_below": hist,
                              "work_share_switched": round(float(w[d < thr].sum() / w.sum()), 4),
                              "h_ms": round(float(np.median(ts)), 4), "rel_diff_vs_all_dmma": rel}), flush=True)
        gp.set_option(_abi.KBG_OPT_SPARSE_DFMA, 0)


if __name__ == "__main__":
    main(sys.argv[1:] or ["sweep56_100Ry", "cubic56_200Ry", "sweep56_400Ry"])

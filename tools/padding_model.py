"""DMMA padding model of the rho / H task structure (CPU, from the oracle index).

Counts the DMMA flops the persistent kernels execute per pass and splits the
overhead over the algorithmic half-count sum_r m(r)^2 (rho and H exploit the
ci <= cj symmetry) into row (M), orbital (K) and point (N) padding.
python tools/padding_model.py [config] [group_rows]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from paper_1402_4247_b200.system import Fe3O4  # noqa: E402


def groups(norb, gr):
    out, cur, first = [], 0, 0
    for c, n in enumerate(norb):
        if cur and cur + n > gr:
            out.append((first, c, cur))
            cur, first = 0, c
        cur += n
        if cur >= gr:
            out.append((first, c + 1, cur))
            cur, first = 0, c + 1
    if cur:
        out.append((first, len(norb), cur))
    return out


def groups_straddle(norb, gr):
    """Row groups of exactly gr orbitals over the concatenated covers (last one shorter)."""
    row0 = np.concatenate([[0], np.cumsum(norb)])
    tot = int(row0[-1])
    out = []
    for r0 in range(0, tot, gr):
        r1 = min(tot, r0 + gr)
        c0 = int(np.searchsorted(row0, r0, side="right") - 1)
        c1 = int(np.searchsorted(row0, r1, side="left"))
        out.append((c0, c1, r1 - r0))
    return out


def popc(x):
    return bin(int(x)).count("1")


def octets(m):
    return [((m >> (8 * i)) & 0xFF) != 0 for i in range(8)]


def quads(m):
    return [((m >> (4 * i)) & 0xF) != 0 for i in range(16)]


def main(cfg="cubic56_200Ry", gr=16, straddle=False):
    f = Fe3O4.config(cfg)
    ix = Oracle(f.system).build_index()
    sp_norb = [s.norb for s in f.system.species]
    spc = f.system.species_of_atom
    alg = ix["sum_m2"] / 2
    r = dict(exec=0.0, exactM=0.0, exactK=0.0, exactN=0.0)
    h = dict(exec=0.0, exactM=0.0, exactN=0.0, exactK=0.0, trimDiag=0.0)
    r["trimDiag"] = 0.0
    nb = ix["nblock"]
    sample = range(0, nb, max(1, nb // 600))
    alg_s = 0.0
    for b in sample:
        c0, c1 = ix["blk_ptr"][b], ix["blk_ptr"][b + 1]
        atoms = ix["cov_atom"][c0:c1]
        masks = [int(m) for m in ix["cov_mask"][c0:c1]]
        norb = [sp_norb[spc[a]] for a in atoms]
        m = np.zeros(64)
        for c, mk in enumerate(masks):
            for p in range(64):
                if (mk >> p) & 1:
                    m[p] += norb[c]
        alg_s += (m * m).sum() / 2
        for (g0, g1, rows) in (groups_straddle(norb, gr) if straddle else groups(norb, gr)):
            tm = (rows + 7) // 8
            for cj in range(g0, len(masks)):
                um = 0
                for ci in range(g0, min(g1, cj + 1)):
                    um |= masks[ci] & masks[cj]
                if not um:
                    continue
                noct = sum(octets(um))
                ks = (norb[cj] + 3) // 4
                nk = ((norb[cj] + 15) // 16) * 16 if ks > 4 else ks * 4
                r["exec"] += tm * 8 * noct * 8 * ks * 4
                r["exactM"] += rows * noct * 8 * ks * 4
                r["exactK"] += tm * 8 * noct * 8 * norb[cj]
                r["exactN"] += tm * 8 * popc(um) * ks * 4
                nq = sum(quads(um))
                # rows of the group's covers ci <= cj only (in-group partners trim the tile)
                rows_le = sum(norb[c] for c in range(g0, min(g1, cj + 1)))
                tm_t = (rows_le + 7) // 8
                r["trimDiag"] += tm_t * 8 * noct * 8 * ks * 4
                h["trimDiag"] += tm_t * 8 * ((norb[cj] + 7) // 8) * 8 * nq * 4
                h["exec"] += tm * 8 * ((norb[cj] + 7) // 8) * 8 * nq * 4
                h["exactM"] += rows * ((norb[cj] + 7) // 8) * 8 * nq * 4
                h["exactN"] += tm * 8 * norb[cj] * nq * 4
                h["exactK"] += tm * 8 * ((norb[cj] + 7) // 8) * 8 * popc(um)
    sc = alg / alg_s
    print(f"{cfg} group_rows={gr} straddle={straddle}: sampled {len(sample)} blocks; algorithmic half-count {alg:.4g} MAC")
    for k, v in r.items():
        print(f"  rho {k:7s} {v * sc / alg:6.3f} x algorithmic")
    for k, v in h.items():
        print(f"  H   {k:7s} {v * sc / alg:6.3f} x algorithmic")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cubic56_200Ry", int(sys.argv[2]) if len(sys.argv) > 2 else 16,
         len(sys.argv) > 3 and sys.argv[3] == "straddle")

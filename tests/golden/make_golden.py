"""Independent numpy restatement of the grid pass -> golden fixtures.

The reference (arxiv/paper_1402_4247) ships no code, test or vector for the
grid path (parity unpinned), so these fixtures come from a
second, independently written implementation of the definitions in
include/kbgrid.h: vectorised numpy over grid points, pair lookups via dicts,
tables tabulated here in numpy. The C++ oracle (oracle/) and the CUDA library
must both reproduce them (tests/test_golden.py, tests/test_gpu_golden.py).

Run: python tests/golden/make_golden.py   (writes tests/golden/*.npz)
"""
from __future__ import annotations

import itertools
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C00, C1, C20, C22, C2 = (0.28209479177387814, 0.4886025119029199, 0.31539156525252005,
                         0.5462742152960396, 1.0925484305920792)


def radial_table(l, alpha, rc, ntab):
    r = np.linspace(0.0, rc, ntab)
    g = 1.0 - (r / rc) ** 2
    e = np.exp(-alpha * r * r)
    u = e * g ** 3
    du = e * (-2 * alpha * r) * g ** 3 + e * 3 * g ** 2 * (-2 * r / rc ** 2)
    # normalise int R^2 r^2 dr with a fine Simpson rule
    x = np.linspace(0.0, rc, 20001)
    gx = 1.0 - (x / rc) ** 2
    f = x ** (2 * l + 2) * (np.exp(-alpha * x * x) * gx ** 3) ** 2
    h = x[1] - x[0]
    integral = h / 3 * (f[0] + f[-1] + 4 * f[1:-1:2].sum() + 2 * f[2:-1:2].sum())
    n = 1.0 / np.sqrt(integral)
    tab = np.stack([n * u, n * du], axis=1)
    tab[-1] = 0.0
    return tab


def slot_of(li, lj, lk):
    return ((((li >> 1) * 2 + (lj >> 1)) * 2 + (lk >> 1)) * 8) + ((li & 1) * 2 + (lj & 1)) * 2 + (lk & 1)


def orbitals(species, d):
    """d: [n,3] displacements inside the sphere -> [n, norb]."""
    l_list, rc, tab = species["l"], species["rc"], species["table"]
    ntab = tab.shape[1]
    d2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
    r = np.sqrt(d2)
    h = rc / (ntab - 1)
    x = r / h
    k = np.minimum(x.astype(np.int64), ntab - 2)
    t = x - k
    omt = 1 - t
    h00, h10, h01, h11 = (1 + 2 * t) * omt * omt, t * omt * omt, t * t * (3 - 2 * t), t * t * (t - 1)
    cols = []
    dx, dy, dz = d[:, 0], d[:, 1], d[:, 2]
    for rad, l in enumerate(l_list):
        T = tab[rad]
        u = h00 * T[k, 0] + h10 * h * T[k, 1] + h01 * T[k + 1, 0] + h11 * h * T[k + 1, 1]
        if l == 0:
            cols.append(C00 * u)
        elif l == 1:
            cols += [C1 * dx * u, C1 * dy * u, C1 * dz * u]
        else:
            cols += [C20 * (2 * dz * dz - dx * dx - dy * dy) * u, C22 * (dx * dx - dy * dy) * u, C2 * dx * dy * u,
                     C2 * dx * dz * u, C2 * dy * dz * u]
    return np.stack(cols, axis=1)


def norb(species):
    return sum(2 * l + 1 for l in species["l"])


def restate(lattice, grid, tau, spc, species):
    A = np.asarray(lattice, dtype=np.float64).reshape(3, 3)
    N = np.asarray(grid)
    npts = int(N.prod())
    nblk = (N + 3) // 4
    ii, jj, kk = np.meshgrid(np.arange(N[0]), np.arange(N[1]), np.arange(N[2]), indexing="ij")
    ii, jj, kk = ii.reshape(-1), jj.reshape(-1), kk.reshape(-1)  # point order p = (i*N1+j)*N2+k
    fi, fj, fk = ii / N[0], jj / N[1], kk / N[2]
    r = np.stack([(fi * A[0, c] + fj * A[1, c]) + fk * A[2, c] for c in range(3)], axis=1)
    blk = ((ii // 4) * nblk[1] + jj // 4) * nblk[2] + kk // 4
    slot = np.array([slot_of(a & 3, b & 3, c & 3) for a, b, c in zip(ii, jj, kk)])
    Ainv = np.linalg.inv(A)
    natom = len(tau)
    # covers: brute-force image search over a generous range
    nR = int(np.ceil(max(s["rc"] for s in species) * np.abs(Ainv).sum(0).max())) + 2
    covers = {}  # block -> list of (atom, R, mask)
    phi = {}  # (atom, R) -> (point indices, values)
    for a in range(natom):
        sp = species[spc[a]]
        for R in itertools.product(range(-nR, nR + 1), repeat=3):
            t = np.array([tau[a][c] + ((R[0] * A[0, c] + R[1] * A[1, c]) + R[2] * A[2, c]) for c in range(3)])
            d = r - t
            d2 = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
            inside = np.nonzero(d2 < sp["rc"] * sp["rc"])[0]
            if len(inside) == 0:
                continue
            phi[(a, R)] = (inside, orbitals(sp, d[inside]))
            for b in np.unique(blk[inside]):
                sel = inside[blk[inside] == b]
                m = 0
                for s in slot[sel]:
                    m |= 1 << int(s)
                covers.setdefault(int(b), []).append((a, R, m))
    nblock = int(nblk.prod())
    blk_ptr = [0]
    cov_atom, cov_R, cov_mask = [], [], []
    for b in range(nblock):
        lst = sorted(covers.get(b, []), key=lambda x: (x[0], x[1]))
        for a, R, m in lst:
            cov_atom.append(a)
            cov_R.append(R)
            cov_mask.append(m)
        blk_ptr.append(len(cov_atom))
    # pairs, canonical-orientation distance test
    def canonical(a, b, R):
        return a < b if a != b else tuple(R) >= (0, 0, 0)

    pairs = []
    nP = int(np.ceil(2 * max(s["rc"] for s in species) * np.abs(Ainv).sum(0).max())) + 2
    for a in range(natom):
        for b in range(natom):
            for R in itertools.product(range(-nP, nP + 1), repeat=3):
                aa, bb, RR = (a, b, R) if canonical(a, b, R) else (b, a, tuple(-x for x in R))
                t = [tau[bb][c] + ((RR[0] * A[0, c] + RR[1] * A[1, c]) + RR[2] * A[2, c]) for c in range(3)]
                d = [t[c] - tau[aa][c] for c in range(3)]
                s = species[spc[aa]]["rc"] + species[spc[bb]]["rc"]
                if (d[0] * d[0] + d[1] * d[1]) + d[2] * d[2] < s * s:
                    pairs.append((a, b, R))
    pairs.sort()
    pid = {p: i for i, p in enumerate(pairs)}
    off = [0]
    for a, b, R in pairs:
        off.append(off[-1] + norb(species[spc[a]]) * norb(species[spc[b]]))
    nnz = off[-1]
    mirror = [pid[(b, a, tuple(-x for x in R))] for a, b, R in pairs]
    # inputs
    rng = np.random.default_rng(1402)
    dm = np.zeros(nnz)
    for p, (a, b, R) in enumerate(pairs):
        if canonical(a, b, R):
            na, nb = norb(species[spc[a]]), norb(species[spc[b]])
            blkv = rng.uniform(-1, 1, size=(na, nb))
            if a == b and R == (0, 0, 0):
                blkv = np.triu(blkv) + np.triu(blkv, 1).T
            dm[off[p]:off[p + 1]] = blkv.reshape(-1)
    for p, (a, b, R) in enumerate(pairs):
        if not canonical(a, b, R):
            q = mirror[p]
            na, nb = norb(species[spc[a]]), norb(species[spc[b]])
            dm[off[p]:off[p + 1]] = dm[off[q]:off[q + 1]].reshape(nb, na).T.reshape(-1)
    veff = np.cos(2 * np.pi * fi) + 0.5 * np.sin(2 * np.pi * (fj + fk)) - 0.3
    dV = abs(np.linalg.det(A)) / npts
    # rho and H by the plain definition over ordered image pairs
    rho = np.zeros(npts)
    h = np.zeros(nnz)
    keys = list(phi.keys())
    for (a, Ra) in keys:
        ia, va = phi[(a, Ra)]
        for (b, Rb) in keys:
            ib, vb = phi[(b, Rb)]
            common, xa, xb = np.intersect1d(ia, ib, assume_unique=True, return_indices=True)
            if len(common) == 0:
                continue
            R = tuple(Rb[c] - Ra[c] for c in range(3))
            p = pid[(a, b, R)]
            na, nb = va.shape[1], vb.shape[1]
            D = dm[off[p]:off[p + 1]].reshape(na, nb)
            fa, fb = va[xa], vb[xb]
            rho[common] += np.einsum("pi,ij,pj->p", fa, D, fb)
            h[off[p]:off[p + 1]] += (fa.T @ (fb * (veff[common] * dV)[:, None])).reshape(-1)
    return {
        "blk_ptr": np.array(blk_ptr, dtype=np.int32), "cov_atom": np.array(cov_atom, dtype=np.int32),
        "cov_R": np.array(cov_R, dtype=np.int32).reshape(-1, 3), "cov_mask": np.array(cov_mask, dtype=np.uint64),
        "pair_a": np.array([p[0] for p in pairs], dtype=np.int32),
        "pair_b": np.array([p[1] for p in pairs], dtype=np.int32),
        "pair_R": np.array([p[2] for p in pairs], dtype=np.int32).reshape(-1, 3),
        "pair_off": np.array(off, dtype=np.int64), "pair_mirror": np.array(mirror, dtype=np.int32),
        "dm": dm, "veff": veff, "dV": dV, "rho": rho, "h": h,
    }


CASES = {
    # orthorhombic cell, grid not a multiple of 4 (ragged blocks), one atom on a grid point
    "dimer_ortho": dict(
        lattice=[[9.0, 0, 0], [0, 10.0, 0], [0, 0, 11.0]], grid=[14, 15, 17],
        tau=[[0.0, 0.0, 0.0], [3.1, 2.2, 4.05]], spc=[0, 1]),
    # triclinic cell, three atoms, one straddling the boundary
    "trimer_triclinic": dict(
        lattice=[[8.0, 0.4, 0.0], [1.1, 7.5, 0.3], [0.2, -0.6, 8.5]], grid=[12, 13, 12],
        tau=[[0.5, 0.4, 0.3], [7.9, 3.0, 2.0], [3.3, 6.6, 7.7]], spc=[0, 1, 1]),
}


def species_defs():
    fe = {"l": [0, 0, 1, 1, 2], "rc": 4.0, "alpha": [0.35, 1.1, 0.4, 0.9, 0.7]}
    ox = {"l": [0, 0, 1, 1], "rc": 3.5, "alpha": [0.45, 1.3, 0.5, 1.2]}
    out = []
    for s in (fe, ox):
        tab = np.stack([radial_table(l, al, s["rc"], 96) for l, al in zip(s["l"], s["alpha"])])
        out.append({"l": s["l"], "rc": s["rc"], "table": tab})
    return out


def main():
    species = species_defs()
    for name, c in CASES.items():
        res = restate(c["lattice"], c["grid"], np.array(c["tau"]), c["spc"], species)
        payload = {k: v for k, v in res.items()}
        payload.update(lattice=np.array(c["lattice"], dtype=np.float64), grid=np.array(c["grid"]),
                       tau=np.array(c["tau"]), spc=np.array(c["spc"], dtype=np.int32))
        for i, s in enumerate(species):
            payload[f"sp{i}_l"] = np.array(s["l"], dtype=np.int32)
            payload[f"sp{i}_rc"] = np.array(s["rc"])
            payload[f"sp{i}_table"] = s["table"]
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **payload)
        print(name, "covers", len(res["cov_atom"]), "pairs", len(res["pair_a"]), "nnz", len(res["dm"]),
              "rho sum", res["rho"].sum() * res["dV"])


if __name__ == "__main__":
    main()

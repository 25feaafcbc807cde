"""Per-opcode instruction and stall-sample breakdown of one kernel from an ncu report (--set full,
--import-source on): python tools/sass_profile.py REPORT.ncu-rep KERNEL_SUBSTRING [top]

Prints warp-level instructions executed per opcode (and per DMMA), and the warp-stall samples
attributed to each opcode -- which instructions the kernel spends its issue slots and its waits on.
"""
import collections
import csv
import io
import subprocess
import sys


def load(path, kname):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows, hdr, take, seen = [], None, False, False
    for row in csv.reader(io.StringIO(out)):
        if row and row[0] == "Kernel Name":
            if seen:
                break  # first matching launch only
            take = kname in row[1]
            hdr = None
            continue
        if not take:
            continue
        if hdr is None:
            hdr = row
            seen = True
            continue
        rows.append(dict(zip(hdr, row)))
    return rows


def main(path, kname, top=25):
    rows = load(path, kname)
    inst = collections.Counter()
    stall = collections.Counter()
    for r in rows:
        op = r["Source"].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1] if len(op) > 1 else o
        o = o.split(".")[0]
        inst[o] += int(r.get("Instructions Executed") or 0)
        stall[o] += int(r.get("Warp Stall Sampling (All Samples)") or 0)
    tot = sum(inst.values())
    dmma = inst.get("DMMA", 0)
    stot = sum(stall.values())
    print(f"{kname}: {tot:,} warp instructions, {dmma:,} DMMA ({tot / max(dmma, 1):.1f} per DMMA), {stot:,} stall samples")
    for o, n in inst.most_common(int(top)):
        print(f"  {o:10s} {n:14,d} {n / max(dmma, 1):6.2f}/DMMA  stalls {stall[o] / max(stot, 1) * 100:5.1f} %")


if __name__ == "__main__":
    main(*sys.argv[1:])


def hot(path, kname, n=200):
    """The hottest straight-line region: instructions executed >= 1/3 of the most executed DMMA."""
    rows = load(path, kname)
    mx = max(int(r.get("Instructions Executed") or 0) for r in rows if "DMMA" in r["Source"])
    for r in rows:
        c = int(r.get("Instructions Executed") or 0)
        if c >= mx / 3:
            print(f'{r["Address"][-5:]} {c:10,d} {int(r.get("Warp Stall Sampling (All Samples)") or 0):5d}  {r["Source"].strip()}')

"""Per CUDA source line: warp instructions executed and warp-stall samples of one kernel, from an ncu
report captured with --import-source on (-lineinfo build):
python tools/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTRING [top]"""
import csv
import io
import subprocess
import sys


def main(path, kname, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fpath, fname, hdr, lines = None, None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            fpath, hdr = r[1], None
            continue
        if r and r[0] == "Function Name":
            fname = r[1]
            continue
        if fname is None or kname not in fname:
            continue
        if hdr is None:
            hdr = r
            ii, si = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if len(r) > ii and r[2] == "-":  # a CUDA source row (SASS rows carry an address)
            try:
                lines.append((int(r[ii]), int(r[si]), fpath.rsplit("/", 1)[-1] + ":" + r[0], r[1].strip()[:100]))
            except ValueError:
                pass
    tot = sum(x[0] for x in lines) or 1
    st = sum(x[1] for x in lines) or 1
    print(f"{kname}: {tot / 1e6:.1f} M warp instructions, {st} stall samples")
    for x in sorted(lines, reverse=True)[:int(top)]:
        print(f"{x[2]:<22} {x[0] / 1e6:7.2f}M {100 * x[0] / tot:5.1f}%  stalls {100 * x[1] / st:5.1f}%  {x[3]}")


if __name__ == "__main__":
    main(*sys.argv[1:])

"""Dynamic SASS opcode mix of one kernel from an `ncu --set full` report (executed warp instructions per
opcode, and the stall samples charged to them).  Usage: python tools/sass_dyn.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    inst = collections.Counter()
    samp = collections.Counter()
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].startswith("0x"):
            d = dict(zip(hdr, r))
            op = d["Source"].strip()
            if op.startswith("@"):
                op = op.split(None, 1)[1]
            op = op.split()[0] if op else "?"
            inst[op] += float(d["Instructions Executed"] or 0)
            samp[op] += float(d["Warp Stall Sampling (All Samples)"] or 0)
    ti, ts = sum(inst.values()), sum(samp.values())
    print(f"total warp instructions {ti:.4e}, stall samples {ts:.0f}")
    for op, v in inst.most_common(top):
        print(f"{op:28s} {v / ti * 100:6.2f} % inst  {samp[op] / ts * 100:6.2f} % samples")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)

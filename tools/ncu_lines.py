"""Per-source-line hot spots of an `ncu --set full --import-source on` report (CUDA view):
warp-stall samples, executed warp instructions and excessive shared-memory wavefronts.
Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    recs = []
    fname = ""
    for r in rows:
        if len(r) >= 2 and r[0] == "File Name":
            fname = r[1].split("/")[-1]
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0].isdigit():
            d = dict(zip(hdr[2:], r[2:]))
            d["Source"] = r[1]
            def f(k):
                try:
                    return float(d.get(k, "0").replace(",", "") or 0)
                except ValueError:
                    return 0.0
            recs.append((fname, int(r[0]), d["Source"].strip()[:90], f("Warp Stall Sampling (All Samples)"),
                         f("Instructions Executed"), f("L1 Wavefronts Shared Excessive"), f("L1 Wavefronts Shared")))
    tot_s = sum(x[3] for x in recs) or 1
    tot_i = sum(x[4] for x in recs) or 1
    tot_x = sum(x[5] for x in recs) or 1
    print(f"total samples {tot_s:.0f}, warp instr {tot_i:.3e}, excessive smem wavefronts {tot_x:.3e}")
    for key, name in ((3, "stall samples"), (4, "instructions"), (5, "excess smem wavefronts")):
        print(f"--- top lines by {name}")
        for x in sorted(recs, key=lambda x: -x[key])[:top]:
            print(f"{x[0]}:{x[1]:5d} samp {x[3] / tot_s:6.1%} inst {x[4] / tot_i:6.1%} xs {x[5] / tot_x:6.1%}  {x[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

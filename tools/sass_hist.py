"""SASS opcode histogram of the hot kernels (cuobjdump -sass on the in-tree objects): the evidence that the
E/M kernels are Blackwell-native (tcgen05 LDTM/STTM, UTCHMMA, UTMALDG/UBLKCP, packed FFMA2/FADD2/FMUL2).
Usage: python tools/sass_hist.py > profiles/r02_sass_hist.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2204_04754_b200", "build")
KERNELS = [("k_fft2.o", "k_fft_em2ILi32ELb1ELi2E"), ("k_fft.o", "k_fft_emILi32ELb1ELi2ELb1ELb0ELi256E"), ("k_fft.o", "k_fft_emILi32ELb1ELi2ELb1ELb0ELi384E"),
           ("k_fft128.o", "k_fft_em128ILb1ELb1E"), ("k_fft_tail.o", "k_fft_tailILb0E"),
           ("k_gemm_tma.o", "gemmt10k_gemm_tma"), ("k_gemm_tma.o", "k_gemm_tma_acc64")]
WATCH = ["FFMA2", "FADD2", "FMUL2", "FFMA", "FADD", "FMUL", "MUFU", "SHFL", "LDS", "STS", "LDG", "STG", "LDL", "STL",
         "LDTM", "STTM", "UTCHMMA", "UTCBAR", "UTMALDG", "UBLKCP", "LDGSTS", "SYNCS", "BAR", "DFMA", "DADD"]


def main():
    for obj, key in KERNELS:
        path = os.path.join(OBJ, obj)
        if not os.path.exists(path):
            continue
        out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
        blocks = re.split(r"\n\s*Function : ", out)
        for b in blocks[1:]:
            name = b.split("\n", 1)[0].strip()
            if key not in name:
                continue
            ops = collections.Counter()
            for line in b.splitlines():
                m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
                if m:
                    ops[m.group(2)] += 1
            tot = sum(ops.values())
            print(f"{obj}: {name[:110]}\n  total {tot} instructions")
            print("  " + ", ".join(f"{k} {ops[k]}" for k in WATCH if ops[k]))
            print("  top: " + ", ".join(f"{k} {v}" for k, v in ops.most_common(14)))
            break


if __name__ == "__main__":
    sys.exit(main())

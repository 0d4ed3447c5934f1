#!/usr/bin/env python3
"""SASS instruction histogram of the hot kernels of libsts_b200.so (cuobjdump -sass):
the evidence that the stencils are TMA (UTMALDG) + mbarrier (SYNCS) pipelines doing FP64
(DFMA / DADD / DMUL) work, and their static instruction counts.

  python tools/sass_histogram.py [lib.so] > profiles/<round>_sass_histogram.md
"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1610_01265_b200/libsts_b200.so"
# (kernel, template args) -> the class name of bench.py / DESIGN.md section 5.2
HOT = {
    r"aniso_tma_kernelILi6ELb1ELb1E": "aniso_pcg_m (merged PCG, full tiles, fused reduction)",
    r"aniso_tma_kernelILi7ELb1ELb0E": "aniso_rkl2_dstage (deviation-form RKL2 stage)",
    r"iso_tma_kernelILi6ELi3ELb1ELb1E": "iso_pcg_m (merged PCG, 3 components)",
    r"iso_tma_kernelILi7ELi3ELb1ELb0E": "iso_rkl2_dstage (deviation-form RKL2 stage, 3 components)",
}
OPS = ["UTMALDG", "UTMASTG", "SYNCS", "DFMA", "DADD", "DMUL", "MUFU", "LDS", "STS", "LDG", "STG", "SHFL",
       "BAR", "FMUL", "IMAD", "BRA"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    print(f"# SASS histogram of the hot kernels (`cuobjdump -sass {LIB}`)\n")
    print("Static instruction counts per kernel (each mnemonic prefix, e.g. SYNCS counts every "
          "SYNCS.* mbarrier op, LDS every shared load).\n")
    print("| kernel | class | total | " + " | ".join(OPS) + " |")
    print("|---|---|---|" + "---|" * len(OPS))
    for f in funcs[1:]:
        name = f.split("\n", 1)[0].strip()
        cls = next((v for k, v in HOT.items() if k in name), None)
        if cls is None:
            continue
        ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(?:\.[\w.]+)?", f)
        c = collections.Counter(ins)
        row = [str(sum(v for k, v in c.items() if k.startswith(op))) for op in OPS]
        print(f"| `{name[:60]}` | {cls} | {len(ins)} | " + " | ".join(row) + " |")


if __name__ == "__main__":
    main()

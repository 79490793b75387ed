#!/usr/bin/env python
"""SASS evidence for the hot kernels (cuobjdump -sass of libtm.so): for each
kernel, the count of every bulk-copy / mbarrier / flag / peer-access mnemonic
that proves the design (UBLKCP = cp.async.bulk on the TMA engine, SYNCS =
mbarrier, LDG/STG .128 = 16-byte accesses, the .STRONG.SYS flag loads and
stores of the cross-rank barriers, REDG = float atomics), followed by the lines
that carry them.  Writes profiles/r02/sass/<kernel>.txt.

    python tools/sass_excerpts.py
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1605_08325_b200", "libtm.so")
OUT = os.path.join(ROOT, "profiles", "r02", "sass")
KERNELS = {
    "tm_direct_tma_kernel_k8_asa16": r"tm_direct_tma_kernelILi8ELb1ELi2048ELi96ELi1E",
    "tm_exchange_tmaws_kernel_k8_asa16_sys": r"tm_exchange_tmaws_kernelILi8ELb1ELb1ELb0E",
    "tm_exchange_tma_kernel_k8_asa16_gpu": r"tm_exchange_tma_kernelILi8ELb1ELb0ELb0E",
    "tm_exchange_oneshot_kernel_k8_asa16_sys": r"tm_exchange_oneshot_kernelILi8ELb1ELb1ELb0E",
    "easgd_round_tma_kernel_n8": r"easgd_round_tma_kernelILi8E",
    "easgd_kernel_mode3_cas128": r"easgd_kernelILi3E",
    "tm_exchange_ll_kernel_k8_asa16_sys": r"tm_exchange_ll_kernelILi8ELb1ELb1ELb0E",
    "tm_exchange_ll2_kernel_k8_asa16_sys": r"tm_exchange_ll2_kernelILi8ELb1ELb1ELb0E",
}
PATTERNS = ["UBLKCP", "SYNCS", "LDG.E.128", "LDG.E.EL.128", "LDG.E.STRONG.GPU.128", "STG.E.128", "STG.E.EF.128",
            "STRONG.SYS", "STRONG.GPU", "FENCE", "MEMBAR", "REDG", "ATOMG", "BAR.SYNC", "F2FP.F16", "HADD2.F32",
            "FADD", "FMUL", "NANOSLEEP", "CS2R", "CAS.128", "LDG.E.128.STRONG.SYS", "STG.E.128.STRONG.SYS"]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    os.makedirs(OUT, exist_ok=True)
    for name, pat in KERNELS.items():
        body = next((f for f in funcs if re.match(r"\S*" + pat, f)), None)
        if body is None:
            print(f"{name}: not found", file=sys.stderr)
            continue
        lines = [l for l in body.splitlines() if re.search(r"/\*[0-9a-f]{4}\*/", l)]
        cnt = collections.Counter()
        for l in lines:
            for p in PATTERNS:
                if p in l:
                    cnt[p] += 1
        keep = [l.strip() for l in lines if any(p in l for p in ("UBLKCP", "SYNCS", "STRONG.SYS", "FENCE", "MEMBAR"))]
        with open(os.path.join(OUT, name + ".txt"), "w") as f:
            f.write(f"# {body.splitlines()[0].strip()}\n# {len(lines)} SASS instructions\n")
            f.write("# mnemonic counts: " + ", ".join(f"{p} {cnt[p]}" for p in PATTERNS if cnt[p]) + "\n\n")
            f.write("\n".join(keep[:400]) + "\n")
        print(name, dict(cnt))


if __name__ == "__main__":
    main()

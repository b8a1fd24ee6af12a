#!/usr/bin/env python
"""Static SASS check of a match-set scan instantiation: the main loop's length
and whether its four row loads issue back to back.

    python tools/loop_stats.py paper_1312_4188_b200/libpfw.so 'ms_scan_kernelILi0ELi8ELi4ELb0ELb0'
"""
import re
import subprocess
import sys


def main(lib, pat):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)
    for f in funcs:
        name = f.split("\n", 1)[0]
        if pat not in name:
            continue
        ins = []
        for line in f.splitlines():
            m = re.match(r"\s*/\*([0-9a-f]{4})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        ldg = [i for i, (a, t) in enumerate(ins) if "LDG.E.128.CONSTANT" in t]
        # the main loop: the last run of 4 LDG.128 within 8 instructions of each other
        for k in range(len(ldg) - 4, -1, -1):
            if ldg[k + 3] - ldg[k] <= 8:
                first = ins[ldg[k]][0]
                together = ldg[k + 3] - ldg[k]
                break
        else:
            print(name[:120], "no 4-load group found")
            continue
        for a, t in ins:
            m = re.search(r"BRA (0x[0-9a-f]+)", t)
            if a > first and m and int(m.group(1), 16) <= first:
                head = int(m.group(1), 16)
                print(f"{name[:110]}: loop {(a - head) // 16 + 1} instrs, 4 row loads within {together} slots")
                break


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])

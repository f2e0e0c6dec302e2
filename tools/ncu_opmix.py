"""Executed-instruction mix by SASS opcode for one kernel of an ncu report (source page)."""
import collections
import csv
import subprocess
import sys


def main(rep, kernel_regex, top="20"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kernel_regex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    mix = collections.Counter()
    for r in rows[2:]:
        src = r[col["Source"]].strip().split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") else src[0]
        try:
            mix[op] += float(r[col["Instructions Executed"]] or 0)
        except ValueError:
            pass
    tot = sum(mix.values()) or 1
    print(f"total warp instructions {tot:.3e}")
    for op, v in mix.most_common(int(top)):
        print(f"  {op:28s} {v:.3e}  {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])

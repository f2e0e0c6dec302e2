"""Per-SASS-instruction stall attribution from an ncu report (source page): the instructions
with the most samples of a given stall reason, and the reason totals by opcode."""
import collections
import csv
import subprocess
import sys


def load(rep, kernel_regex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kernel_regex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    return hdr, rows[2:]


def main(rep, kernel_regex, reason="stall_long_sb", top="25"):
    top = int(top)
    hdr, rows = load(rep, kernel_regex)
    col = {h: i for i, h in enumerate(hdr)}
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]

    def val(r, h):
        try:
            return float(r[col[h]] or 0)
        except ValueError:
            return 0.0

    tot = collections.Counter()
    by_op = collections.defaultdict(collections.Counter)
    for r in rows:
        op = r[col["Source"]].strip().split()[0] if r[col["Source"]].strip() else "?"
        if op.startswith("@"):
            op = r[col["Source"]].strip().split()[1]
        op = op.split(".")[0]
        for h in reasons:
            v = val(r, h)
            tot[h] += v
            by_op[h][op] += v
    all_s = sum(tot.values()) or 1
    print("reason totals:", ", ".join(f"{h[6:]}={100 * v / all_s:.1f}%" for h, v in tot.most_common(10)))
    for h in (reason,):
        print(f"{h} by opcode:", ", ".join(f"{op}={100 * v / all_s:.1f}%" for op, v in by_op[h].most_common(8)))
    print(f"top instructions by {reason}:")
    best = sorted(rows, key=lambda r: -val(r, reason))[:top]
    for r in best:
        print(f"  {val(r, reason):8.0f}  {r[col['Address']][-5:]}  {r[col['Source']].strip()[:90]}")


if __name__ == "__main__":
    main(*sys.argv[1:])

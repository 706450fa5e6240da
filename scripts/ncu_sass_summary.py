"""Summarise an ncu report's SASS source page for one kernel: opcode mix and stall hot spots.

python scripts/ncu_sass_summary.py REPORT.ncu-rep KERNEL_REGEX [top]
"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def main(rep, kre, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    name = lines[0]
    # the page repeats a "Kernel Name" block per matching launch: keep the first
    nxt = next((i for i in range(1, len(lines)) if lines[i].startswith('"Kernel Name"')), len(lines))
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:nxt]))))
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    ops = Counter()
    stall = []
    tot_inst = 0
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
        try:
            n = int(r[ix["Instructions Executed"]] or 0)
        except ValueError:
            continue
        ops[op.split(".")[0]] += n
        tot_inst += n
        stall.append((int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[ix["Address"]], src, n))
    print(name[:150])
    print("warp instructions executed:", tot_inst)
    for op, n in ops.most_common(top):
        print(f"  {op:12s} {n:12d} {100.0 * n / max(tot_inst, 1):5.1f}%")
    tot = sum(s[0] for s in stall)
    print("top stall samples (of", tot, ")")
    for s, a, src, n in sorted(stall, reverse=True)[:top]:
        print(f"  {s:7d} {100.0 * s / max(tot, 1):5.1f}%  {src[:70]:70s} n={n}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)

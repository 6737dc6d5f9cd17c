#!/usr/bin/env python3
"""Summarise an ncu report's SASS source page (warp-stall sampling) per
kernel: instruction-class mix and where the stall samples sit (by opcode and
by stall reason), plus the hottest instruction windows.
  python tools/ncu_sass_profile.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import io
import re
import subprocess
import sys


def pages(rep, kregex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kregex],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'^"Kernel Name",', out, flags=re.M)
    for b in blocks[1:]:
        name, rest = b.split("\n", 1)
        yield name.strip().strip(",").strip('"'), list(csv.reader(io.StringIO(rest)))


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 else "."
    for name, rows in pages(rep, kre):
        hdr = rows[0]
        ix = {h: i for i, h in enumerate(hdr)}
        stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        by_op = collections.Counter()
        samp_op = collections.Counter()
        stall_tot = collections.Counter()
        stall_op = collections.defaultdict(collections.Counter)
        total_inst = 0
        seq = []
        for r in rows[1:]:
            if len(r) < len(hdr):
                continue
            src = r[ix["Source"]].strip()
            op = src.split()[0] if src else "?"
            if op.startswith("@"):
                op = src.split()[1]
            opb = op.split(".")[0]
            n = int(r[ix["Instructions Executed"]] or 0)
            s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            by_op[opb] += n
            samp_op[opb] += s
            total_inst += n
            for h in stall_cols:
                v = int(r[ix[h]] or 0)
                stall_tot[h] += v
                stall_op[opb][h] += v
            seq.append((src, n, s))
        tot_s = sum(samp_op.values()) or 1
        print("=" * 100)
        print(name[:120])
        print("warp-instructions executed %d, stall samples %d" % (total_inst, tot_s))
        print("%-10s %10s %6s %8s  top stalls" % ("opcode", "inst", "inst%", "samp%"))
        for op, n in by_op.most_common(22):
            top = ", ".join("%s %.1f" % (h[6:], 100.0 * v / tot_s) for h, v in stall_op[op].most_common(3) if v)
            print("%-10s %10d %5.1f%% %7.1f%%  %s" % (op, n, 100.0 * n / total_inst, 100.0 * samp_op[op] / tot_s, top))
        print("stall reasons:", ", ".join("%s %.1f%%" % (h[6:], 100.0 * v / tot_s) for h, v in stall_tot.most_common(12)))


if __name__ == "__main__":
    main()

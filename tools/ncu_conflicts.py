#!/usr/bin/env python3
"""Shared-memory wavefronts above ideal per CUDA source line (ncu cuda,sass view).
  python tools/ncu_conflicts.py report.ncu-rep [function-name substring]"""
import collections
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
want = sys.argv[2] if len(sys.argv) > 2 else ""
hdr = fn = kern = cur = None
acc = collections.defaultdict(lambda: [0, 0])
for raw in out.splitlines():
    if not raw.startswith('"'):
        continue
    parts = raw.strip().strip(",")[1:-1].split('","')
    if parts[0] == "File Path":
        fn = parts[1].split("/")[-1]
        continue
    if parts[0] == "Function Name":
        kern = parts[1]
        continue
    if parts[0] == "Line No":
        hdr = parts
        ix = {h: i for i, h in enumerate(hdr)}
        continue
    if hdr is None or want not in (kern or ""):
        continue
    if len(parts) > len(hdr):
        parts = [parts[0], '","'.join(parts[1:len(parts) - len(hdr) + 2])] + parts[len(parts) - len(hdr) + 2:]
    if parts[0] != "":
        cur = (kern[:60], fn, parts[0], parts[1][:70])
        continue
    try:
        w = int(parts[ix["L1 Wavefronts Shared"]])
        wi = int(parts[ix["L1 Wavefronts Shared Ideal"]])
    except (ValueError, KeyError, IndexError):
        continue
    a = acc[cur]
    a[0] += w
    a[1] += wi
for k, (w, wi) in sorted(acc.items(), key=lambda kv: -(kv[1][0] - kv[1][1]))[:12]:
    if w > wi:
        print("%8d excess (%8d / ideal %8d)  %s" % (w - wi, w, wi, " ".join(k[1:])))

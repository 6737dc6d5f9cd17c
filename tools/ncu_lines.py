#!/usr/bin/env python3
"""Per-CUDA-source-line stall attribution from an ncu report (cuda,sass view).
  python tools/ncu_lines.py report.ncu-rep kernel-regex [top] [function-name substring]"""
import subprocess
import sys


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                         capture_output=True, text=True).stdout
    fn = kernel = None
    hdr = None
    acc = {}
    tot = 0
    seen_kernel = None
    for raw in out.splitlines():
        if not raw.startswith('"'):
            continue
        parts = raw.strip().strip(",")[1:-1].split('","')
        if hdr is not None and parts[0] not in ("File Path", "Function Name", "Line No") and len(parts) > len(hdr):
            # the source text held '","': keep the line number and the trailing metric fields
            parts = [parts[0], '","'.join(parts[1:len(parts) - len(hdr) + 2])] + parts[len(parts) - len(hdr) + 2:]
        r = parts
        if not r:
            continue
        if r[0] == "File Path":
            fn = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            if seen_kernel is None and (len(sys.argv) < 5 or sys.argv[4] in r[1]):
                seen_kernel = r[1]
            kernel = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if kernel != seen_kernel or hdr is None or len(r) < len(hdr) or r[0] == "" or r[4] in ("-", ""):
            continue
        s = int(r[4])
        key = (fn, int(r[0]))
        d = acc.setdefault(key, {"src": r[1][:80], "s": 0, "st": {}})
        d["s"] += s
        tot += s
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and r[i] not in ("-", "", "0"):
                d["st"][h[6:]] = d["st"].get(h[6:], 0) + int(r[i])
    print(seen_kernel, "samples", tot)
    for (f, ln), d in sorted(acc.items(), key=lambda kv: -kv[1]["s"])[:top]:
        st = ", ".join("%s %.1f" % (k, 100.0 * v / tot) for k, v in sorted(d["st"].items(), key=lambda kv: -kv[1])[:4])
        print("%5.1f%% %s:%d  %-60s | %s" % (100.0 * d["s"] / tot, f, ln, d["src"].strip()[:60], st))


if __name__ == "__main__":
    main()

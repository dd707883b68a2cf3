#!/usr/bin/env python
"""Per-source-line warp-stall samples of an ncu report (needs -lineinfo and
--import-source on): python tools/ncu_lines.py report.ncu-rep [top]
Prints the lines with the most stall samples, their executed instructions and
the dominant stall reasons."""
import csv
import io
import os
import subprocess
import sys


def main():
    rep, top = os.path.abspath(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, cwd="/tmp").stdout
    rows, fname, hdr, lines = list(csv.reader(io.StringIO(out))), "", None, []
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "" or r[0] == "Function Name":
            continue
        # source text may contain unescaped quotes/commas: index metrics from the end
        nm = len(hdr) - 4
        if len(r) < nm + 2:
            continue
        d = dict(zip(hdr[4:], r[-nm:]))
        r = [r[0], ",".join(r[1:len(r) - nm - 2])]
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            ins = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
                  and v not in ("", "-") and v.isdigit() and int(v) > 0}
        lines.append((s, ins, fname, r[0], r[1].strip()[:90], stalls))
    tot = sum(x[0] for x in lines) or 1
    print(f"total samples {tot}")
    for s, ins, f, ln, src, st in sorted(lines, reverse=True)[:top]:
        top3 = ", ".join(f"{k} {v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print(f"{100.0 * s / tot:5.1f}% {ins:9d} {f}:{ln:5s} {src}  [{top3}]")


if __name__ == "__main__":
    main()

"""Attribute an ncu SASS-page capture to CUDA source lines (build container).

ncu's CUDA-source page needs the source imported at capture time; the SASS
page does not.  This joins `ncu -i REP --page source --csv --print-source sass`
with `nvdisasm -g` line info of the same cubin and prints the top source lines
by executed warp instructions and by stall samples.

    python profiles/sass_lines.py REP.ncu-rep CUBIN MANGLED_KERNEL_NAME [top]
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def line_map(cubin, kernel):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    sec = out.split(f".text.{kernel}:", 1)[1].split("//---------------------", 1)[0]
    cur = "?"
    m = {}
    for ln in sec.splitlines():
        f = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if f and "inlined at" not in ln:
            cur = f"{f.group(1).rsplit('/', 1)[-1]}:{f.group(2)}"
            continue
        a = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if a:
            m[int(a.group(1), 16)] = cur
    return m


def main():
    rep, cubin, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lm = line_map(cubin, kernel)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, ie, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    base = int(rows[2][ia], 16)
    inst, samp = defaultdict(int), defaultdict(int)
    tot_i = tot_s = 0
    for r in rows[2:]:
        if len(r) <= ie or not r[ia].startswith("0x"):
            continue
        off = int(r[ia], 16) - base
        key = lm.get(off, "?")
        i, s = int(r[ie] or 0), int(r[isamp] or 0)
        inst[key] += i
        samp[key] += s
        tot_i += i
        tot_s += s
    print(f"total warp instructions {tot_i}, stall samples {tot_s}")
    print(f"{'line':24s} {'inst%':>7s} {'samples%':>9s}")
    for k, v in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{k:24s} {100.0 * v / tot_i:7.2f} {100.0 * samp[k] / max(tot_s, 1):9.2f}")


if __name__ == "__main__":
    main()

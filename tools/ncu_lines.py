#!/usr/bin/env python
"""Per-source-line profile of one kernel: ncu's per-SASS-instruction metrics (``ncu -i rep
--page source --csv --print-source=sass``) mapped to CUDA source lines through the cubin's line
table (``nvdisasm --print-line-info``).  Prints the lines with the most stall samples and
executed instructions.

    python tools/ncu_lines.py REP.ncu-rep OBJ.o KERNEL_SUBSTR [--mangled MANGLED] [--top 40]
"""
import argparse
import collections
import csv
import io
import os
import re
import subprocess
import tempfile


def line_table(obj, mangled):
    with tempfile.TemporaryDirectory() as d:
        subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d,
                              stdout=subprocess.DEVNULL)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        dis = subprocess.check_output(["nvdisasm", "--print-line-info", os.path.join(d, cub)], text=True)
    lines = dis.split("\n")
    st = next(i for i, x in enumerate(lines) if x.strip() == mangled + ":")
    off2line, cur = {}, None
    for x in lines[st + 1:]:
        if re.match(r"^(_Z\w+|\.nv\.\S+):$", x.strip()):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', x)
        if m:
            if cur is None:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+", x)
        if m:
            if cur:
                off2line[int(m.group(1), 16)] = cur
            cur = None
    return off2line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("obj")
    ap.add_argument("kernel")
    ap.add_argument("--mangled", required=True)
    ap.add_argument("--top", type=int, default=40)
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', out)
    blk = next(b for b in blocks[1:] if args.kernel in b.split("\n", 1)[0])
    rows = list(csv.reader(io.StringIO(blk.split("\n", 1)[1])))
    h, data = rows[0], [r for r in rows[1:] if len(r) > 5]
    ia, iss = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    iex, ith = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
    off2line = line_table(args.obj, args.mangled)
    base = int(data[0][ia], 16)
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    last = None
    for r in data:
        key = off2line.get(int(r[ia], 16) - base, last)
        last = key
        a = agg[key]
        a[0] += float(r[iss] or 0)
        a[1] += float(r[iex] or 0)
        a[2] += float(r[ith] or 0)
    ts = sum(a[0] for a in agg.values()) or 1
    te = sum(a[1] for a in agg.values()) or 1
    tt = sum(a[2] for a in agg.values()) or 1
    print(f"warp instructions {te:.4g}, thread instructions {tt:.4g}, samples {ts:.4g}")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][0])[: args.top]:
        print(f"{str(k):32s} stall {a[0] / ts:6.3f}  warp-instr {a[1] / te:6.3f}  thread-instr {a[2] / tt:6.3f}  "
              f"threads/instr {a[2] / max(a[1], 1):5.1f}")


if __name__ == "__main__":
    main()

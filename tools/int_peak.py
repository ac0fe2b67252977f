#!/usr/bin/env python
"""Measure the B200's integer-instruction issue ceiling for the LPT bin-loop mix (tools/int_peak.cu)
and write it as the ALU roofline denominator bench.py uses (``--out``, default
profiles/r02/int_peak.json).

    python tools/int_peak.py [--out profiles/r02/int_peak.json]   (on the GPU box)

Per kernel: the loop body's SASS instructions are counted from ``cuobjdump -sass`` (ptxas may fuse
or split the PTX ops, so the source count is not used), and thread-instructions per second =
body instructions x iterations x threads / CUDA-event time, best of 5 at full occupancy.  SM clocks
and throttle reasons are sampled by nvidia-smi during the runs."""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import re
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "int_peak.cu")
LIB = os.path.join(HERE, "libintpeak.so")
KINDS = {0: "mix_pack", 1: "iadd3", 2: "imnmx", 3: "lop3", 4: "isetp_sel"}
KERNEL_SASS = {0: "k_mix_pack", 1: "k_singleILi0E", 2: "k_singleILi1E", 3: "k_singleILi2E", 4: "k_singleILi3E"}


def build(force=False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(SRC) > os.path.getmtime(LIB):
        nvcc = "/usr/local/cuda/bin/nvcc"
        subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
                               "-Xcompiler", "-fPIC", "-shared", SRC, "-o", LIB])
    return LIB


def loop_bodies() -> dict:
    """SASS instructions of each kernel's main loop (the largest backward branch's body) and the
    mnemonic histogram of that body."""
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], text=True)
    out = {}
    for part in re.split(r"\n\s*Function : ", sass)[1:]:
        name = part.split("\n", 1)[0]
        ins = []
        for line in part.split("\n"):
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        best = None
        for addr, txt in ins:
            b = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", txt)
            if b and int(b.group(1), 16) < addr:
                body = [t for a, t in ins if int(b.group(1), 16) <= a <= addr]
                if best is None or len(body) > len(best):
                    best = body
        if best is None:
            continue
        hist = {}
        for t in best:
            op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
            hist[op] = hist.get(op, 0) + 1
        for k, key in KERNEL_SASS.items():
            if key in name:
                out[k] = {"instructions": len(best), "mnemonics": hist}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "int_peak.json"))
    ap.add_argument("--iters", type=int, default=20000)
    args = ap.parse_args()
    import torch

    sys.path.insert(0, ROOT)
    from bench import ClockSampler

    build()
    bodies = loop_bodies()
    L = C.CDLL(LIB)
    L.int_peak_launch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_void_p, C.c_void_p]
    L.int_peak_launch.restype = C.c_int
    torch.cuda.set_device(0)
    props = torch.cuda.get_device_properties(0)
    sms = props.multi_processor_count
    blocks = sms * 8  # 8 CTAs x 256 threads = 2048 threads per SM (full occupancy)
    out = torch.empty(blocks * 256, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    clk = ClockSampler(0)
    clk.start()
    time.sleep(0.3)
    res = {}
    for kind, name in KINDS.items():
        for _ in range(2):  # warm-up
            assert L.int_peak_launch(kind, blocks, args.iters, 12345, out.data_ptr(), stream.cuda_stream) > 0
        best = None
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            L.int_peak_launch(kind, blocks, args.iters, 12345, out.data_ptr(), stream.cuda_stream)
            b.record(stream)
            b.synchronize()
            ms = a.elapsed_time(b)
            best = ms if best is None else min(best, ms)
        body = bodies[kind]
        thread_instr = body["instructions"] * args.iters * blocks * 256
        res[name] = {"ms": best, "loop_sass_instructions": body["instructions"], "mnemonics": body["mnemonics"],
                     "thread_instr_per_s": thread_instr / (best / 1000.0),
                     "per_sm_per_clk": None}
    clocks = clk.stop()
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    for r in res.values():
        r["per_sm_per_clk"] = r["thread_instr_per_s"] / (sms * mhz * 1e6)
    line = {
        "what": "integer thread-instruction issue ceiling, full occupancy (148 SMs x 8 CTAs x 256 threads), "
                "8 independent chains per thread; loop-body SASS instructions counted from cuobjdump",
        "gpu": props.name, "sms": sms, "clocks": clocks, "iters": args.iters,
        "peak_gops": res["mix_pack"]["thread_instr_per_s"] / 1e9,
        "peak_kind": "mix_pack (VIADD, LOP3, VIMNMX, ISETP, SEL, predicated VIADD: the k_pack_lanes bin step)",
        "nominal_gops": sms * 128 * mhz * 1e6 / 1e9,
        "kernels": res,
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(line, f, indent=1)
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())

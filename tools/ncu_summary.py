#!/usr/bin/env python
"""Summarise an ncu --set full capture: key metrics per kernel, the hottest SASS, and
(optionally) merge per-launch DRAM traffic into profiles/ncu_summary.json (read by bench.py).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json profiles/ncu_summary.json] [--top 30]
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
from pathlib import Path

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.per_cycle_active",
    "smsp__warps_eligible.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_per_inst_issued.ratio", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_fma.sum",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__cycles_active.sum",
]


POLICY = {"0": "MCSF", "1": "MCBENCH", "2": "ALPHA", "3": "ALPHA_BETA"}


def abi_name(short: str) -> str:
    """ncu's demangled template name -> the name sched_last_kernel() reports."""
    m = re.match(r"k_mc_(lane|flat)<(\d), (\d+)(?:, (\d))?>", short)
    if m:
        return f"k_mc_{m.group(1)}<{POLICY[m.group(2)]}" + (",p16>" if m.group(4) == "1" else ">")
    m = re.match(r"k_mc_small<(\d), (\d), (\d)>", short)
    if m:
        pol, multi, qreg = m.groups()
        tags = [POLICY[pol]] + ([] if multi == "1" else ["per-round"]) + ([] if qreg == "1" else ["smemq"])
        return "k_mc_small<" + ",".join(tags) + ">"
    m = re.match(r"k_ring<(\d)>", short)
    if m:
        return f"k_ring<{POLICY[m.group(1)]}>"
    return short


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep: str) -> list[dict]:
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_units"] = dict(zip(hdr, units))
        out.append(d)
    return out


def to_bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def to_ns(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    return x * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)


def alu_inst(d: dict):
    try:
        pct = float(d["sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active"].replace(",", ""))
        cyc = float(d["sm__cycles_active.sum"].replace(",", ""))
    except (KeyError, ValueError):
        return None
    return pct / 100.0 * 2.0 * cyc


def hot_sass(rep: str, top: int):
    text = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass")
    rows = list(csv.reader(io.StringIO(text)))
    if len(rows) < 3:
        return [], 0
    hdr = rows[1]
    ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    ist = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[ia] or 0), int(r[ist] or 0), r[isrc].strip()))
        except (IndexError, ValueError):
            continue
    tot = sum(d[0] for d in data)
    return sorted(data, key=lambda x: -x[1])[:top], tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--json")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    kernels = {}
    for d in raw(a.rep):
        name = d.get("Kernel Name", "?")
        short = re.sub(r"\(.*", "", name).replace("void ", "").replace("kv::", "")
        u = d["_units"]
        rd = to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
        wr = to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        dur = to_ns(d["gpu__time_duration.sum"], u["gpu__time_duration.sum"])
        print(f"== {short}  ({abi_name(short)})")
        for m in METRICS:
            if m in d:
                print(f"  {m:70s} {d[m]:>16s} {u.get(m, '')}")
        print(f"  dram bytes per launch: {rd + wr:.4g}  duration {dur / 1e6:.4f} ms")
        kernels[abi_name(short)] = {"ncu_name": short, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                          "duration_ms": dur / 1e6, "source": Path(a.rep).name,
                          "issue_active_pct": d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                          "registers": d.get("launch__registers_per_thread"),
                          "warp_inst": d.get("smsp__inst_executed.sum"),
                          # ALU-pipe warp instructions: ncu's percentage of the pipe's peak
                          # (0.5 warp-inst / clk / SMSP = 2 / clk / SM) x active SM cycles
                          "alu_inst": alu_inst(d),
                          "fma_inst": d.get("sm__inst_executed_pipe_fma.sum"),
                          "alu_pipe_pct": d.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active")}
    hot, tot = hot_sass(a.rep, a.top)
    print(f"== hottest SASS by stall samples (total warp instructions {tot:.4g})")
    for c, s, src in hot:
        print(f"  {c:12d} {s:7d}  {src[:90]}")
    if a.json:
        p = Path(a.json)
        cur = json.loads(p.read_text()) if p.exists() else {"kernels": {}}
        cur.setdefault("kernels", {}).update(kernels)
        cur["note"] = ("dram bytes per launch from ncu --set full --clock-control none (one launch per "
                       "kernel, cold cache, replayed); see the .txt summaries beside this file")
        p.write_text(json.dumps(cur, indent=1))


if __name__ == "__main__":
    main()

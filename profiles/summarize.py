"""Summarise ncu captures into the committed, per-round profile notes.

    python profiles/summarize.py gpurun_out/prof.ncu-rep [launches.csv] > profiles/rNN_<name>.md
    python profiles/summarize.py --traffic gpurun_out/prof.ncu-rep > profiles/rNN_traffic.json
    python profiles/summarize.py --inst gpurun_out/prof.ncu-rep > profiles/rNN_inst.json

For every kernel launch in the report: duration, DRAM bytes read/written,
DRAM / SM throughput, IPC, occupancy, registers, per-pipe utilisation, L2
atomic sectors, the warp-stall mix and the hottest source lines (needs
-lineinfo + --import-source). With a launch-list CSV (the
``--metrics gpu__time_duration.sum`` pass) it also prints each kernel's share
of the step. ``--traffic`` writes {kernel: dram bytes per launch}, which
bench.py reports as ``roofline.traffic``.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import Counter, defaultdict

RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "smsp__inst_executed.sum",
       "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
       "lts__t_requests_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_red.sum.per_second",
       "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "lts__t_sector_hit_rate.pct")

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
              "us": 1e-6, "ms": 1e-3, "s": 1.0,
              "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def raw_rows(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for n, u, v in zip(hdr, units, r):
            d[n] = (v, u)
        out.append(d)
    return out


def val(d, name):
    v, u = d.get(name, ("", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * UNIT_SCALE.get(u, 1.0)


def source_lines(rep, kernel_id, top=12):
    txt = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
              "--launch-skip", str(kernel_id), "--launch-count", "1")
    rows = list(csv.reader(io.StringIO(txt)))
    out, fname, hdr = [], None, None
    stalls = Counter()
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit():
            continue

        def num(n):
            x = r[hdr.index(n)] if n in hdr else ""
            return int(x) if x.isdigit() else 0

        ie = num("Instructions Executed")
        st = num("Warp Stall Sampling (All Samples)")
        for n, x in zip(hdr, r):
            if n.startswith("stall_") and "Not Issued" not in n and x.isdigit():
                stalls[n[6:]] += int(x)
        if ie or st:
            out.append((ie, st, f"{fname}:{r[0]}", r[1].strip()[:80]))
    ti = sum(o[0] for o in out) or 1
    ts = sum(o[1] for o in out) or 1
    lines = [f"| {100 * ie / ti:4.1f}% | {100 * st / ts:4.1f}% | `{loc}` | `{src}` |"
             for ie, st, loc, src in sorted(out, reverse=True)[:top]]
    tot = sum(stalls.values()) or 1
    mix = ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in stalls.most_common(6))
    return lines, mix


def launches(csv_path):
    rows = list(csv.reader(open(csv_path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = ["| kernel | launches | avg us | share |", "|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | "
                   f"{100 * sum(v) / tot:.1f}% |")
    return out


def main():
    if sys.argv[1] == "--traffic":
        traffic = {}
        for d in raw_rows(sys.argv[2]):
            name = d.get("Kernel Name", ("", ""))[0].split("(")[0].split("<")[0].replace(
                "void ", "").replace("fvv::", "")
            b = (val(d, "dram__bytes_read.sum") or 0) + (val(d, "dram__bytes_write.sum") or 0)
            traffic.setdefault(name, []).append(b)
        print(json.dumps({k: sum(v) / len(v) for k, v in traffic.items()}, indent=1))
        return
    if sys.argv[1] == "--facts":
        # per kernel, averaged over its launches in the capture: what bench.py
        # needs to put each kernel against its own roofline (DRAM bytes, warp
        # instructions, FP64 thread operations, L2 RED requests per launch)
        facts = {}
        for d in raw_rows(sys.argv[2]):
            name = d.get("Kernel Name", ("", ""))[0].split("(")[0].split("<")[0].replace(
                "void ", "").replace("fvv::", "")
            cyc = val(d, "sm__cycles_elapsed.avg") or 0
            fp64 = sum((val(d, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum."
                                "per_cycle_elapsed") or 0) for op in ("dadd", "dmul", "dfma"))
            f = {"duration_s": val(d, "gpu__time_duration.sum"),
                 "dram_bytes": (val(d, "dram__bytes_read.sum") or 0) +
                               (val(d, "dram__bytes_write.sum") or 0),
                 "warp_inst": val(d, "smsp__inst_executed.sum"),
                 "fp64_thread_ops": fp64 * cyc,
                 "fp64_pipe_pct_active": val(d, "sm__pipe_fp64_cycles_active.avg."
                                                "pct_of_peak_sustained_active"),
                 "l2_red_requests": val(d, "lts__t_requests_srcunit_tex_op_red.sum"),
                 "ipc_active": val(d, "sm__inst_executed.avg.per_cycle_active")}
            facts.setdefault(name, []).append(f)
        out = {}
        for k, v in facts.items():
            out[k] = {n: (sum(x[n] for x in v if x[n] is not None) / len(v)
                          if any(x[n] is not None for x in v) else None) for n in v[0]}
            out[k]["launches_captured"] = len(v)
        print(json.dumps(out, indent=1))
        return
    if sys.argv[1] == "--inst":
        inst = {}
        for d in raw_rows(sys.argv[2]):
            name = d.get("Kernel Name", ("", ""))[0].split("(")[0].split("<")[0].replace(
                "void ", "").replace("fvv::", "")
            inst.setdefault(name, []).append(val(d, "smsp__inst_executed.sum") or 0)
        print(json.dumps({k: sum(v) / len(v) for k, v in inst.items()}, indent=1))
        return
    rep = sys.argv[1]
    print(f"# ncu summary: `{rep}`\n")
    if len(sys.argv) > 2:
        print("## Launch list (gpu__time_duration per launch, serialised; see file for cache mode)\n")
        print("\n".join(launches(sys.argv[2])) + "\n")
    for i, d in enumerate(raw_rows(rep)):
        name = d.get("Kernel Name", ("?", ""))[0]
        print(f"## [{i}] `{name}`\n")
        dur = val(d, "gpu__time_duration.sum")
        rd, wr = val(d, "dram__bytes_read.sum"), val(d, "dram__bytes_write.sum")
        print(f"- duration {dur * 1e6:.1f} us; DRAM read {rd / 1e6:.1f} MB, write {wr / 1e6:.1f} MB "
              f"({(rd + wr) / dur / 1e9:.0f} GB/s)")
        for n in RAW[3:]:
            x = val(d, n)
            if x is not None:
                print(f"- `{n}` = {x:,.2f}")
        try:
            lines, mix = source_lines(rep, i)
            print(f"- warp-stall mix: {mix}\n")
            print("| inst | stall | line | source |\n|---|---|---|---|")
            print("\n".join(lines))
        except subprocess.CalledProcessError:
            pass
        print()


if __name__ == "__main__":
    main()

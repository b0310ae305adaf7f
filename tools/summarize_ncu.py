"""Summarise ncu captures into profiles/ (tracked).

  python tools/summarize_ncu.py <round> <launches.csv> <rep>... 

Writes profiles/ncu_<round>_launches.txt (per-kernel launch count, total and
mean device time and share of the captured step -- cold-cache, serialised, so
compare shares), profiles/ncu_<round>_<kernel>.txt (key --set full metrics per
launch) and updates profiles/ncu_traffic.json (dram bytes read+write per
launch for each kernel, read by bench.py for the roofline "traffic" field).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__sass_inst_executed_op_global_ld.sum", "smsp__sass_inst_executed_op_global_st.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
]
STALLS = "smsp__pcsamp_warps_issue_stalled_"


def short(name):
    for k in ("k_perm", "k_tile", "k_fact", "k_gate1q", "k_controlled", "k_cut_phase", "k_tree_wide", "k_tree",
              "k_marginals", "k_exchange_peer", "k_swap_peer", "k_swap_local", "k_fill",
              "k_gaussian", "k_scale", "k_pair_halves"):
        if k in name:
            return k
    return name[:40]


def launches(rnd, path):
    rows = list(csv.reader(open(path)))
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            body = rows[i + 1:]
            break
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("Metric Unit"))
    agg = defaultdict(list)
    for r in body:
        if len(r) == len(hdr) and r[mi] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", ""))
            unit = r[ui]
            ms = v / 1e6 if unit == "ns" else (v / 1e3 if unit in ("us", "usecond") else v)
            agg[short(r[ki])].append(ms)
    total = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list, round {rnd}: {os.path.basename(path)}",
             "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised;",
             "#   compare shares, not absolute times)",
             f"{'kernel':18s} {'launches':>8s} {'total_ms':>10s} {'mean_ms':>9s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k:18s} {len(v):8d} {sum(v):10.3f} {sum(v)/len(v):9.4f} {sum(v)/total:7.1%}")
    out = os.path.join(PROF, f"ncu_{rnd}_launches.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rnd, rep):
    if rep.endswith(".raw.csv"):  # exported on the GPU box (ncu -i rep --page raw --csv)
        raw = open(rep).read().splitlines()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout.splitlines()
    # capture tag (r02b_qaoa.raw.csv -> qaoa): pool-mode captures get their own
    # traffic keys (k_fact@qaoa), the config-2 sweep keeps the bare kernel name
    tag = os.path.basename(rep).split(".")[0].split("_", 1)[-1]
    suffix = "" if tag in ("fact", "tile", "other", rnd) else "@" + tag
    rows = list(csv.reader(raw))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    name_i = idx.get("Kernel Name")
    traffic_path = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    per_kernel = defaultdict(list)
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        k = short(r[name_i]) + suffix
        rec = {}
        for key in KEYS:
            if key in idx and r[idx[key]] not in ("", "n/a"):
                rec[key] = (r[idx[key]], units[idx[key]])
        st = {h[len(STALLS):]: float(r[i]) for h, i in idx.items()
              if h.startswith(STALLS) and not h.endswith("not_issued") and r[i] not in ("", "n/a")}
        tot = sum(st.values()) or 1.0
        rec["stalls (share of pc samples)"] = (
            " ".join(f"{k2}={v / tot:.2f}" for k2, v in sorted(st.items(), key=lambda kv: -kv[1])[:6]),
            "")
        per_kernel[k].append(rec)
    for k, recs in per_kernel.items():
        lines = [f"# ncu --set full, round {rnd}: {os.path.basename(rep)}, kernel {k}"]
        tb = []
        for i, rec in enumerate(recs):
            lines.append(f"launch {i}:")
            for key, (v, u) in rec.items():
                lines.append(f"  {key:62s} {v:>16s} {u}" if u or len(v) < 17 else f"  {key}: {v}")
            try:
                rd = float(rec["dram__bytes_read.sum"][0].replace(",", ""))
                wr = float(rec["dram__bytes_write.sum"][0].replace(",", ""))
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                tb.append(rd * scale[rec["dram__bytes_read.sum"][1]] +
                          wr * scale[rec["dram__bytes_write.sum"][1]])
            except (KeyError, ValueError):
                pass
        open(os.path.join(PROF, f"ncu_{rnd}_{k}.txt"), "w").write("\n".join(lines) + "\n")
        if tb:
            amps = AMPS.get(os.path.basename(rep)) or AMPS.get(tag)
            traffic[k] = {"bytes_per_launch": sum(tb) / len(tb), "launches": len(tb),
                          "amplitudes_per_launch": amps,
                          "bytes_per_amplitude": (sum(tb) / len(tb) / amps) if amps else None,
                          "source": os.path.basename(rep), "round": rnd,
                          "note": "dram read+write per launch from the ncu capture; bench.py "
                                  "scales bytes_per_amplitude to its own launch size"}
        print("\n".join(lines[:30]))
    json.dump(traffic, open(traffic_path, "w"), indent=1)


AMPS = {}

if __name__ == "__main__":
    rnd = sys.argv[1]
    for a in sys.argv[2:]:
        if a.startswith("--amps="):  # --amps=<rep basename>:<log2 amplitudes>
            name, lg = a[len("--amps="):].split(":")
            AMPS[name] = 1 << int(lg)
            continue
        if a.endswith(".csv") and not a.endswith(".raw.csv"):
            launches(rnd, a)
        else:
            full(rnd, a)

"""Summarise an ncu report (--set full) into profiles/: per-kernel speed-of-light,
DRAM bytes, L2 hit rate, issue utilisation, SM-active vs elapsed cycles and
the top warp-stall reasons; and refresh profiles/traffic.json.

    python tools/ncu_summary.py gpurun_out/seq_full.ncu-rep profiles/r02_seq_full_summary.txt
    python tools/ncu_summary.py gpurun_out/seq_4k.ncu-rep profiles/r02_seq_4k_summary.txt "one 4K RGB frame" traffic_4k.json
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration", 1e-3, "us"),
    ("smsp__inst_executed.sum", "warp_instructions", 1.0, ""),
    ("dram__bytes_read.sum", "dram_read", None, ""),
    ("dram__bytes_write.sum", "dram_write", None, ""),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct", 1.0, "%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct", 1.0, "%"),
    ("sm__warps_active.avg.per_cycle_active", "warps_active_per_sm", 1.0, ""),
    ("sm__cycles_active.avg", "sm_active_cycles", 1.0, ""),
    ("gpc__cycles_elapsed.max", "elapsed_cycles", 1.0, ""),
    ("launch__registers_per_thread", "registers", 1.0, ""),
    ("launch__grid_size", "grid", 1.0, ""),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_pct", 1.0, "%"),
]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6,
        "ns": 1.0, "us": 1e3, "ms": 1e6}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def short(name):
    base = name.split("(")[0]
    return base.replace("void ", "")


def main(rep, out_txt, what="one 1080p RGB frame", traffic_name="traffic.json"):
    h, units, rows = raw(rep)
    lines, kern = [], []
    for r in rows:
        d = {"kernel": short(r[h.index("Kernel Name")])}
        for k, nm, sc, _ in KEYS:
            if k not in h:
                continue
            v, u = r[h.index(k)], units[h.index(k)]
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            if nm.startswith("dram"):
                x *= UNIT.get(u, 1.0)
            elif nm == "duration":
                x = x * UNIT.get(u, 1.0) / 1e3  # -> us
            d[nm] = x
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), k.split("stalled_")[1].split("_per_issue")[0]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        d["top_stalls_cycles_per_issue"] = {n: round(v, 3) for v, n in stalls[:6]}
        kern.append(d)
    for d in kern:
        sa = d.get("sm_active_cycles", 0) / max(1.0, d.get("elapsed_cycles", 1))
        lines.append(
            f"{d['kernel']:<58s} {d.get('duration', 0):7.2f} us  inst {d.get('warp_instructions', 0) / 1e6:6.2f} M  "
            f"DRAM r/w {d.get('dram_read', 0) / 1e6:6.2f}/{d.get('dram_write', 0) / 1e6:5.2f} MB  "
            f"L2 hit {d.get('l2_hit_pct', 0):5.1f}%  issue {d.get('issue_active_pct', 0):5.1f}%  "
            f"warps/SM {d.get('warps_active_per_sm', 0):5.2f}  SM-active/elapsed {sa:4.2f}  regs {d.get('registers', 0):.0f}")
        lines.append("    stalls (cycles per issued instruction): "
                     + ", ".join(f"{k} {v}" for k, v in d["top_stalls_cycles_per_issue"].items()))
    hdr = (f"# ncu --set full summary of {os.path.basename(rep)} ({what}'s pass sequence, "
           "--cache-control none: warm L2 as in the real sequence, --clock-control none)\n")
    with open(out_txt, "w") as fh:
        fh.write(hdr + "\n".join(lines) + "\n")
    print(hdr + "\n".join(lines))
    # traffic.json: mean DRAM bytes and instructions per launch of the dominant kernels
    agg = {}
    for d in kern:
        k = d["kernel"]
        if "k_row_roll" in k:
            tag = "k_row_roll_it" if ", 1, " in k else "k_row_roll_f0"
            agg.setdefault(tag, []).append(d)
            continue
        if "k_col" in k:
            tag = "k_col2" if "k_col2" in k else "k_col3" if "k_col3" in k else "k_col"
        else:
            tag = ("k_row_it" if ", 1>" in k or k.endswith("1>") else
                   "k_row_f0" if k.endswith("0>") else "k_row_fin" if k.endswith("3>") else None)
        if tag is None:
            continue
        agg.setdefault(tag, []).append(d)
    tj = {"note": "dram__bytes_read.sum + dram__bytes_write.sum and smsp__inst_executed.sum per launch, mean over "
                  f"the launches in {os.path.basename(rep)} (ncu --set full --cache-control none, warm L2)"}
    for tag, ds in agg.items():
        n = len(ds)
        tj[tag] = {"bytes": sum(x.get("dram_read", 0) + x.get("dram_write", 0) for x in ds) / n,
                   "warp_instructions": sum(x.get("warp_instructions", 0) for x in ds) / n,
                   "duration_us": sum(x.get("duration", 0) for x in ds) / n,
                   "issue_active_pct": sum(x.get("issue_active_pct", 0) for x in ds) / n,
                   "launches": n, "source": out_txt}
    with open(os.path.join(os.path.dirname(out_txt), traffic_name), "w") as fh:
        json.dump(tj, fh, indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])

"""Summarise `ncu --set full` captures of the SpMV kernel into profiles/.

    python tools/ncu_summarize.py CONFIG REPORT.ncu-rep|RAW.csv [ROUND_TAG]

Writes profiles/<tag>_ncu_<config>.csv (the key metrics, one row per
kernel) and merges {config: {...}} into profiles/ncu_summary.json, which
bench.py reads for roofline.traffic (DRAM bytes per launch).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1, "ms": 1, "nsecond": 1e-6}


def main():
    cfg, rep = sys.argv[1], sys.argv[2]
    tag = sys.argv[3] if len(sys.argv) > 3 else "r01"
    if rep.endswith(".csv"):  # `ncu -i REP --page raw --csv` exported on the GPU box
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out_rows = []
    for r in data:
        name = r[hdr.index("Kernel Name")]
        rec = {"kernel": name}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                v = float(r[i].replace(",", "") or 0)
                u = units[i]
                if k.startswith("dram__bytes"):
                    v *= SCALE.get(u, 1)
                if k == "gpu__time_duration.sum":
                    v *= SCALE.get(u, 1)  # -> ms
                rec[k] = v
        out_rows.append(rec)
    path = os.path.join(ROOT, "profiles", f"{tag}_ncu_{cfg}.csv")
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=["kernel"] + [k for k in KEYS if k in hdr])
        w.writeheader()
        w.writerows(out_rows)
    main_k = [r for r in out_rows if "k_spmv_stream" in r["kernel"]] or out_rows
    k = main_k[-1]
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    rd, wr = k.get("dram__bytes_read.sum", 0), k.get("dram__bytes_write.sum", 0)
    summ[cfg] = {"kernel": k["kernel"][:160], "dram_bytes_per_launch": int(rd + wr),
                 "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
                 "gpu_time_ms_ncu": round(k.get("gpu__time_duration.sum", 0), 4),
                 "warp_instructions": int(k.get("smsp__inst_executed.sum", 0)),
                 "issue_active_pct": round(k.get(
                     "smsp__issue_active.avg.pct_of_peak_sustained_active", 0), 1),
                 "source": f"profiles/{tag}_ncu_{cfg}.csv (ncu --set full --clock-control none)"}
    with open(summ_path, "w") as fh:
        json.dump(summ, fh, indent=1)
    print(json.dumps(summ[cfg], indent=1))


if __name__ == "__main__":
    main()

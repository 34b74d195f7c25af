"""Turns the ncu outputs under gpurun_out/ into the committed summaries under profiles/.

  gpurun_out/launches_batch.csv, launches_single.csv : `ncu --metrics gpu__time_duration.sum` launch lists
  gpurun_out/prof_dmma.ncu-rep, prof_single.ncu-rep  : `ncu --set full` captures of the two hot kernels
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")
SRC = os.path.join(ROOT, "gpurun_out")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"


def launch_summary(name):
    path = os.path.join(SRC, name)
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            hdr, rows = r, rows[i + 1:]
            break
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for r in rows:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = r[ki].split("(")[0].replace("void ", "")
        tot[k] = tot.get(k, 0.0) + float(r[vi].replace(",", ""))
        cnt[k] += 1
    total = sum(tot.values())
    return [{"kernel": k, "launches": cnt[k], "total_us": v / 1e3, "avg_us": v / 1e3 / cnt[k], "share": v / total}
            for k, v in sorted(tot.items(), key=lambda kv: -kv[1])]


KEYS = ["gpu__time_duration.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]


def full_summary(rep):
    path = os.path.join(SRC, rep)
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append({"kernel": d.get("Kernel Name"), **{k: f"{d[k]} {u[k]}".strip() for k in KEYS if k in d}})
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    summary = {}
    prefix = sys.argv[2] if len(sys.argv) > 2 else ""      # e.g. "s2_": files of a later session
    for name in (prefix + "launches_batch.csv", prefix + "launches_single.csv"):
        if os.path.exists(os.path.join(SRC, name)):
            summary[name] = launch_summary(name)[:12]
    for rep in sorted(f for f in os.listdir(SRC) if f.startswith(prefix + "prof_") and f.endswith(".ncu-rep")):
        summary[rep] = full_summary(rep)
    json.dump(summary, open(os.path.join(OUT, f"{TAG}_ncu_summary.json"), "w"), indent=1)
    # per-launch DRAM traffic of the dominant batched kernel, for bench.py's roofline.traffic
    dm = prefix + "prof_dmma.ncu-rep"
    if dm in summary and summary[dm]:
        def to_bytes(s):
            v, unit = s.split()[0].replace(",", ""), s.split()[1] if len(s.split()) > 1 else "byte"
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return float(v) * mult
        recs = summary[dm]
        traffic = sum(to_bytes(r["dram__bytes_read.sum"]) + to_bytes(r["dram__bytes_write.sum"]) for r in recs) / len(recs)
        json.dump({"dram_bytes_per_launch": traffic, "captures": len(recs), "source": f"{TAG}_ncu_summary.json"},
                  open(os.path.join(OUT, "dmma_gemm_traffic.json"), "w"), indent=1)
    # per-launch DRAM traffic of the batched round kernel (one launch = one check round of 25 layers)
    rk = prefix + "prof_round.ncu-rep"
    if rk in summary and summary[rk]:
        def to_bytes2(s):
            v, unit = s.split()[0].replace(",", ""), s.split()[1] if len(s.split()) > 1 else "byte"
            return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        recs = summary[rk]
        traffic = sum(to_bytes2(r["dram__bytes_read.sum"]) + to_bytes2(r["dram__bytes_write.sum"]) for r in recs) / len(recs)
        json.dump({"dram_bytes_per_launch": traffic, "captures": len(recs), "launch": "round_kernel, 4096-column rounds (25 layers each)",
                   "source": f"{TAG}_ncu_summary.json"}, open(os.path.join(OUT, "round_kernel_traffic.json"), "w"), indent=1)
    # DRAM bytes per iteration of the streamed single-QP tier (tools/profile_tier1.py runs
    # fixed_iters(100)), for bench.py's roofline_single_qp_stream.traffic
    t1 = prefix + "prof_tier1.ncu-rep"
    if t1 in summary and summary[t1]:
        def to_bytes1(s):
            v, unit = s.split()[0].replace(",", ""), s.split()[1] if len(s.split()) > 1 else "byte"
            return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        r = summary[t1][0]
        json.dump({"dram_bytes_per_iteration": (to_bytes1(r["dram__bytes_read.sum"]) + to_bytes1(r["dram__bytes_write.sum"])) / 100.0,
                   "iterations_in_capture": 100, "source": f"{TAG}_ncu_summary.json"},
                  open(os.path.join(OUT, "stream_traffic.json"), "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()

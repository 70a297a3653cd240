"""Summarise gpurun_out/prof_*.ncu-rep into profiles/<round>/ncu_*_summary.txt
and profiles/ncu_traffic.json (dram bytes per launch, the bench's `traffic`).

usage: python scripts/summarize_ncu.py r01
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dadd_pred_on.sum"]
# report -> (kernel key used by bench.py, config)
REPORTS = {"prof_batch2": ("batch2_rk4_kernel", "C2"),
           "prof_c3": ("chain_tiles_persistent<8,256>", "C3"),
           "prof_c4": ("chain_rk4_kernel<8>", "C4"),
           "prof_dense": ("dense_rk4_gemm", "C5")}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    out_dir = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(out_dir, exist_ok=True)
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for rep, (kernel, cfg) in REPORTS.items():
        path = os.path.join(ROOT, "gpurun_out", rep + ".ncu-rep")
        if not os.path.exists(path):
            continue
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, u, v = rows[0], rows[1], rows[2]
        lines = [f"ncu --set full --clock-control none --import-source on -c 1 ({rep})"]
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"{k:78s} {v[i]} {u[i]}")
        stalls = sorted(((float(v[i]), k) for i, k in enumerate(h)
                         if "smsp__average_warps_issue_stalled" in k
                         and k.endswith("per_issue_active.ratio")), reverse=True)[:6]
        lines.append("top stalls (cycles per issued instruction):")
        lines += [f"  {val:7.3f} {k}" for val, k in stalls]
        open(os.path.join(out_dir, f"ncu_{rep}_summary.txt"), "w").write("\n".join(lines) + "\n")
        rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        traffic.setdefault(kernel, {})[cfg] = (float(v[rd]) * SCALE[u[rd]] +
                                               float(v[wr]) * SCALE[u[wr]])
        print("\n".join(lines))
    json.dump(traffic, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    main()

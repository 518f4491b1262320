"""Summarise a round's GPU artifacts (gpurun_out/) into profiles/ (committed).

    python tools/summarize_profile.py round1

Reads gpurun_out/prof_<tag>.ncu-rep (ncu --set full of block_cells_tmem_kernel
on the bench workload), gpurun_out/launches_<tag>.csv (ncu launch list of the
bench command), gpurun_out/bench_<tag>.json, microbench/bank-probe outputs;
writes profiles/<tag>_*.{txt,json,csv} and profiles/ncu_block_cells_traffic.json
(the per-launch DRAM traffic bench.py reports as roofline.traffic)."""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum", "sm__cycles_elapsed.avg",
]


def ncu_csv(*args):
    r = subprocess.run(["ncu", *args], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    lines = [f"# ncu --set full summary, block_cells_tmem_kernel, tag {tag}",
             "# command: tools/profile_round.sh (ncu --set full --clock-control none -k regex:block_cells_tmem -c 1",
             "#          python tools/prof_block.py 100000)  -- 100k M156 cells, P regime, Jacobi-BiCGSTAB", ""]
    rep = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    metrics = {}
    if os.path.exists(rep):
        rows = ncu_csv("-i", rep, "--page", "raw", "--csv")
        h, u, v = rows[0], rows[1], rows[2]
        d = {h[i]: (u[i], v[i]) for i in range(len(h))}
        instance = d.get("Kernel Name", ("", ""))[1]
        lines.insert(3, f"# instance: {instance}")
        for k in KEYS:
            if k in d:
                lines.append(f"{k:75s} {d[k][1]:>22s} {d[k][0]}")
                metrics[k] = d[k]
        sass = ncu_csv("-i", rep, "--page", "source", "--csv", "--print-source", "sass")
        hdr = sass[1]
        idx = {x: i for i, x in enumerate(hdr)}
        byop, stall = collections.Counter(), collections.Counter()
        tot = samples = 0.0
        for r in sass[2:]:
            if len(r) < len(hdr):
                continue
            ie = float(r[idx["Instructions Executed"]] or 0)
            tot += ie
            src = r[idx["Source"]].split()
            op = (src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else "")).split(".")[0]
            byop[op] += ie
            samples += float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
            for k in hdr:
                if k.startswith("stall_") and "Not Issued" not in k:
                    try:
                        stall[k] += float(r[idx[k]] or 0)
                    except ValueError:
                        pass
        lines += ["", "instruction mix (% of warp instructions):"]
        lines += [f"  {op:12s} {c / tot * 100:5.1f}%" for op, c in byop.most_common(20)]
        lines += ["", "warp stall reasons (% of samples):"]
        lines += [f"  {k:28s} {c / samples * 100:5.1f}%" for k, c in stall.most_common(10)]
        traffic = float(metrics["dram__bytes_read.sum"][1]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[
            metrics["dram__bytes_read.sum"][0]] + float(metrics["dram__bytes_write.sum"][1]) * {
            "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[metrics["dram__bytes_write.sum"][0]]
        with open(os.path.join(PROF, "ncu_block_cells_traffic.json"), "w") as f:
            pct = lambda k: float(metrics[k][1]) / 100.0 if k in metrics else None  # noqa: E731
            json.dump({"kernel": "block_cells_tmem_kernel", "instance": instance, "algorithm": "bicgstab",
                       "species": 156, "cells": 100000, "tag": tag,
                       "dram_bytes_per_launch_scaled": traffic,
                       "shared_pipe_frac": pct("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
                       "issue_active_frac": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                       "fp64_pipe_frac": pct("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                       "shared_ld_wavefronts": float(metrics.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
                                                                 ("", "0"))[1]),
                       "shared_st_wavefronts": float(metrics.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
                                                                 ("", "0"))[1]),
                       "note": "dram__bytes_read.sum + dram__bytes_write.sum of one launch on the bench workload "
                               "(100k M156 cells, P regime); compulsory bytes are 1.496e9; the *_frac are the same "
                               "capture's shared-memory pipe, issue and FP64 utilisation"}, f, indent=1)
    with open(os.path.join(PROF, f"{tag}_ncu_block_cells_tmem.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    for name in (f"launches_{tag}.csv", f"bench_{tag}.json", "microbench_b200.json"):
        if os.path.exists(os.path.join(OUT, name)):
            shutil.copy(os.path.join(OUT, name), os.path.join(PROF, f"{tag}_{name}" if tag not in name else name))
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "round1")

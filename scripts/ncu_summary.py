"""Summarise an ncu report (--set full) into profiles/: key throughput,
occupancy, pipe, DRAM and stall metrics of one kernel launch.

  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_k_assemble_cfg2.txt [--json key]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (ms)"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock (Hz)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active (% of peak)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy (%)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe (SFU: MUFU rsqrt/rcp) % of peak"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % of peak"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % of peak"),
    ("sm__warps_active.avg.per_cycle_active", "active warps / SM"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / block (B)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% of peak)"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "DFMA thread-instructions"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "DMUL thread-instructions"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread-instructions"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    hdr, units, data = raw(rep)
    lines = []
    summary = []
    for r in data:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines.append(f"kernel: {d.get('Kernel Name', '?')[:110]}")
        lines.append(f"grid {d.get('launch__grid_size')} x block {d.get('launch__block_size')}")
        for k, label in KEYS:
            if k in d:
                lines.append(f"  {label:34s} {d[k]} {u.get(k, '')}")
        stalls = []
        for k, v in d.items():
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    stalls.append((float(v), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(s for s, _ in stalls) or 1.0
        lines.append("  warp stall reasons (% of samples): " + ", ".join(
            f"{n} {100 * s / tot:.1f}" for s, n in sorted(stalls, reverse=True)[:7]))
        def num(k):
            try:
                return float(d[k])
            except Exception:
                return None
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        dram = sum((num(k) or 0.0) * scale.get(u.get(k, "byte"), 1.0)
                   for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        summary.append({"kernel": d.get("Kernel Name", ""), "duration_ms": num("gpu__time_duration.sum"),
                        "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                        "xu_pipe_pct": num("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                        "dram_bytes": dram})
        lines.append("")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if "--json" in sys.argv:
        key = sys.argv[sys.argv.index("--json") + 1]
        path = "profiles/ncu_summary.json"
        try:
            allj = json.load(open(path))
        except Exception:
            allj = {}
        allj[key] = {"k_assemble_dram_bytes_per_launch": summary[0]["dram_bytes"], "report": rep,
                     "fp64_pipe_pct": summary[0]["fp64_pipe_pct"], "xu_pipe_pct": summary[0]["xu_pipe_pct"],
                     "duration_ms": summary[0]["duration_ms"]}
        json.dump(allj, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()

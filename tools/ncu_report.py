"""Summarise one kernel launch of an ncu --set full report for profiles/.

    python tools/ncu_report.py <report.ncu-rep> <key> <so_digest> [algorithmic_bytes]

Prints the launch's duration, DRAM traffic (read + write), L2 and L1 traffic
and bandwidth, FMA / ALU / LSU pipe utilisation, issue-active and warp
occupancy, and records the DRAM bytes under <key> in profiles/traffic.json
together with the digest of the library build it was taken on (bench.py
reports roofline.traffic only for a matching build)."""
import csv
import json
import subprocess
import sys
from pathlib import Path

rep, key, digest = sys.argv[1], sys.argv[2], sys.argv[3]
algo = float(sys.argv[4]) if len(sys.argv) > 4 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def num(name):
    v, u = d[name]
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
             "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "second": 1.0}.get(u, 1)
    return x * scale, u


dur, _ = num("gpu__time_duration.sum")
dram = num("dram__bytes_read.sum")[0] + num("dram__bytes_write.sum")[0]
lines = [f"kernel: {d.get('Kernel Name', ('?',))[0]}",
         f"duration: {dur * 1e3:.3f} ms   grid {d['launch__grid_size'][0]} x block {d['launch__block_size'][0]}, "
         f"{d['launch__registers_per_thread'][0]} regs"]
lines.append(f"DRAM read+write per launch: {dram / 1e9:.3f} GB ({dram / dur / 1e9:.0f} GB/s)"
             + (f"; algorithmic {algo / 1e9:.3f} GB (x{dram / algo:.2f})" if algo else ""))
for name, label, scale in (("lts__t_bytes.sum", "L2 traffic", 1), ("lts__t_sectors.sum", "L2 traffic", 32),
                           ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 reads from the SMs", 32),
                           ("l1tex__t_bytes.sum", "L1 traffic", 1),
                           ("SM_B.TriageCompute.l1tex__t_sectors.sum", "L1 traffic", 32)):
    if name in d and d[name][0] != "no data":
        b = num(name)[0] * scale
        lines.append(f"{label} ({name}): {b / 1e9:.1f} GB per launch = {b / dur / 1e12:.2f} TB/s")
for name in ("lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
             "l1tex__throughput.avg.pct_of_peak_sustained_active",
             "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
             "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
             "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
             "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
             "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
             "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
             "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"):
    if name in d:
        lines.append(f"{name}: {d[name][0]} {d[name][1]}")
print("\n".join(lines))
tf = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
data = json.loads(tf.read_text()) if tf.exists() else {}
data[key] = {"dram_bytes": int(dram), "file": Path(rep).name, "so_digest": digest, "duration_ms": dur * 1e3}
if algo:
    data[key]["algorithmic_bytes"] = int(algo)
tf.write_text(json.dumps(data, indent=1) + "\n")

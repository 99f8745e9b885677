"""Summarise an ncu report: key metrics per launch + top stall SASS lines."""
import csv, subprocess, sys, collections

rep = sys.argv[1]
mets = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "sm__cycles_active.avg",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
        "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_wait_per_warp_active.pct",
        "smsp__warp_issue_stalled_no_instruction_per_warp_active.pct"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(mets)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d.get("Kernel Name", "")[:70])
    for m in mets:
        if m in d:
            print(f"   {m:70s} {d[m]}")
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    hh = rows[1]
    ix = {k: i for i, k in enumerate(hh)}
    body = []
    for r in rows[2:]:
        if len(r) < len(hh) or r[0].startswith("Kernel"):
            if body:
                break
            continue
        body.append(r)
    tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
    print("total samples", tot)
    for r in sorted(body, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:int(sys.argv[2])]:
        print(f'{r[ix["Address"]][-5:]} {r[ix["Source"]][:64]:64s} samp={r[ix["Warp Stall Sampling (All Samples)"]]:>5} exec={r[ix["Instructions Executed"]]}')

"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (tracked).

  python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/r1_launches.txt
  python scripts/ncu_summary.py full gpurun_out/prof_gather.ncu-rep profiles/r1_gather_full.txt [traffic_key]
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "pcie__read_bytes.sum", "pcie__write_bytes.sum", "lts__t_sectors_aperture_sysmem_op_read.sum",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_requests_srcunit_ltcfabric.sum",
]
SUBSTR = ["pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"].split("(")[0]
        agg.setdefault(name, []).append(float(d["Metric Value"]))
    total = sum(sum(v) for k, v in agg.items() if "fill_synthetic" not in k)
    with open(dst, "w") as fh:
        fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        fh.write(f"# source: {os.path.basename(src)}; {len(data)} launches; share excludes k_fill_synthetic (setup)\n")
        fh.write(f"{'kernel':45s} {'n':>5s} {'mean_us':>10s} {'min_us':>10s} {'max_us':>10s} {'share':>7s}\n")
        for k, v in agg.items():
            share = "" if "fill_synthetic" in k else f"{100 * sum(v) / total:6.1f}%"
            fh.write(f"{k:45s} {len(v):5d} {sum(v) / len(v) / 1e3:10.2f} {min(v) / 1e3:10.2f} {max(v) / 1e3:10.2f} {share:>7s}\n")
    print(open(dst).read())


def full(src, dst, key=None):
    out = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full --clock-control none; source {os.path.basename(src)}"]
    traffic = []
    for r in rows[2:]:
        lines.append("kernel: " + r[hdr.index("Kernel Name")])
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                lines.append(f"  {m:62s} {r[i]:>16s} {units[i]}")
        for i, h in enumerate(hdr):
            if any(x in h for x in SUBSTR):
                lines.append(f"  {h.split('.', 2)[-1] if h.count('.') > 3 else h:62s} {r[i]:>16s} {units[i]}")
        try:
            ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
            traffic.append(float(r[ir]) * SCALE[units[ir]] + float(r[iw]) * SCALE[units[iw]])
        except (ValueError, KeyError):
            pass
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if key and traffic:
        p = os.path.join(os.path.dirname(dst), "ncu_traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[key] = sum(traffic) / len(traffic)
        json.dump(d, open(p, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](*sys.argv[2:])

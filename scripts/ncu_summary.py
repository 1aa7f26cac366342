#!/usr/bin/env python
"""Summarise an ncu --set full capture (.ncu-rep) into a small JSON for profiles/.

usage: python scripts/ncu_summary.py REPORT.ncu-rep [channel_frames] > profiles/NAME.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
    "lts__t_requests_srcunit_ltcfabric.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__inst_executed.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
]


def main():
    rep = sys.argv[1]
    frames = float(sys.argv[2]) if len(sys.argv) > 2 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                try:
                    d[k] = {"value": float(r[i].replace(",", "")), "unit": units[i]}
                except ValueError:
                    d[k] = {"value": r[i], "unit": units[i]}
        if frames:
            rd = d.get("dram__bytes_read.sum", {})
            wr = d.get("dram__bytes_write.sum", {})
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            try:
                tot = rd["value"] * scale[rd["unit"]] + wr["value"] * scale[wr["unit"]]
                d["dram_bytes_per_channel_frame"] = tot / frames
            except (KeyError, TypeError):
                pass
        out.append(d)
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()

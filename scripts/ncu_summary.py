"""Summarise an ncu --set full report (raw page) into a short text block.

    python scripts/ncu_summary.py gpurun_out/prof_x.ncu-rep [--bytes B]

--bytes: algorithmic bytes of the profiled launch, to print the DRAM
traffic / algorithmic ratio.
"""

import argparse
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 sectors read (tex)"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 sectors write (tex)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "L1 global ld sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "L1 global ld requests"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "warp cycles / issued inst"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--bytes", type=float, default=None)
    a = ap.parse_args()
    launches, units = raw(a.rep)
    for d in launches:
        print(f"kernel: {d.get('Kernel Name', '?')[:100]}")
        for k, name in KEYS:
            if k in d:
                print(f"  {name:32s} {d[k]} {units.get(k, '')}")
        rd = d.get("dram__bytes_read.sum")
        wr = d.get("dram__bytes_write.sum")
        if rd and wr:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = float(rd) * scale.get(units["dram__bytes_read.sum"], 1) + \
                float(wr) * scale.get(units["dram__bytes_write.sum"], 1)
            print(f"  {'dram bytes total':32s} {tot:.4g} B")
            if a.bytes:
                print(f"  {'dram / algorithmic':32s} {tot / a.bytes:.3f}")
        stalls = []
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith(
                    "_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):
                                                -len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  top stalls (warps per issue):",
              ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))


if __name__ == "__main__":
    sys.exit(main())

"""Condense an `ncu --set full` report into profiles/ncu_summary.json.

Maps kernel instantiations to the bench's kernel kinds and records, per
launch: duration, DRAM bytes (read+write), L1 data-pipe / issue utilisation,
sectors and instructions.  bench.py reads `dram_bytes_per_launch` for the
roofline `traffic` field.
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

KIND = [("fp_kernel<<unnamed>::CylGeo, 1", "fp_correction"),
        ("fp_kernel_small<<unnamed>::CylGeo, 1", "fp_correction"),
        ("fp_kernel<<unnamed>::CylGeo, 2", "fp_residual"),
        ("fp_kernel_small<<unnamed>::CylGeo, 2", "fp_residual"),
        ("fp_kernel_small<<unnamed>::CylGeo, 4", "fp_correction_resid"),
        ("bp_kernel<<unnamed>::CylVox, 2", "bp_update"),
        ("pack_gather_cyl", "pack_gather"),
        ("pack_quads", "pack_quads")]

FIELDS = {"duration_ms": ("gpu__time_duration.sum", 1.0),
          "dram_read_bytes": ("dram__bytes_read.sum", None),
          "dram_write_bytes": ("dram__bytes_write.sum", None),
          "l1_data_pipe_pct": ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1.0),
          "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
          "l1_sectors": ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 1.0),
          "instructions": ("smsp__inst_executed.sum", 1.0),
          "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
          "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1.0),
          "registers": ("launch__registers_per_thread", 1.0),
          "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
          "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
          "alu_pipe_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
          "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1.0),
          "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0)}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep, out, label):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(txt.splitlines()))
    h, units, rows = r[0], r[1], r[2:]
    ki = h.index("Kernel Name")
    res = json.loads(Path(out).read_text()) if Path(out).exists() else {}
    res.setdefault("kernels", {})
    res["source"] = label
    for row in rows:
        name = row[ki]
        kind = next((k for pat, k in KIND if pat in name), None)
        if kind is None:
            continue
        d = {"kernel": name[:120]}
        for f, (metric, _) in FIELDS.items():
            if metric in h:
                i = h.index(metric)
                v = float(row[i].replace(",", "")) if row[i] else 0.0
                if f.startswith("dram"):
                    v *= UNIT.get(units[i], 1)
                d[f] = v
        d["dram_bytes_per_launch"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
        res["kernels"][kind] = d
    Path(out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[1])

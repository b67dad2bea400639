"""Condense an `ncu --set full` report into a per-kernel-kind JSON summary.

Maps kernel instantiations to the bench's kernel kinds and records, per
launch: duration, DRAM bytes (read+write), L2 bytes (lts__t_bytes), FMA-pipe
active cycles and its per-SM-cycle peak (derived from the .sum and the
pct_of_peak_sustained_active of the same launch), L1 data-pipe / issue
utilisation, sectors and instructions.  bench.py's roofline reads
profiles/r02_ncu_summary.json (`dram_bytes_per_launch`,
`lts_bytes_per_launch`, `fma_cycles_active_per_launch`,
`fma_cycles_per_sm_cycle`).

Capture with the extra metrics, e.g.
  ncu --set full --metrics lts__t_bytes.sum,sm__pipe_fma_cycles_active.sum,\
      sm__cycles_active.sum --clock-control none --import-source on ...
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

KIND = [("fp_kernel<<unnamed>::CylGeo, 1", "fp_correction"),
        ("fp_kernel<<unnamed>::CylGeo, 4", "fp_correction_resid"),
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
          "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
          "lts_bytes": ("lts__t_bytes.sum", None),
          "l2_throughput_pct": ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", 1.0),
          "l1tex_throughput_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1.0),
          "fma_cycles_active_sum": ("sm__pipe_fma_cycles_active.sum", 1.0),
          "sm_cycles_active_sum": ("sm__cycles_active.sum", 1.0),
          "sm_mhz": ("sm__cycles_elapsed.avg.per_second", None),
          "sm_cycles_elapsed_avg": ("sm__cycles_elapsed.avg", 1.0),
          "l1_wavefronts_avg_per_sm": ("l1tex__data_pipe_lsu_wavefronts.avg", 1.0),
          "fmaheavy_pipe_pct": ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
                                1.0)}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(rep, out, label):
    if rep.endswith(".csv"):                 # the raw page already exported on the box
        txt = Path(rep).read_text()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
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
            # some metrics carry a section prefix ("SM_A.TriageCompute.<metric>")
            cands = [j for j, n in enumerate(h) if n == metric or n.endswith("." + metric)]
            if cands:
                i = cands[0]
                v = float(row[i].replace(",", "")) if row[i] else 0.0
                if f.startswith("dram") or f == "lts_bytes":
                    v *= UNIT.get(units[i], 1)
                if f == "sm_mhz":
                    v *= {"hz": 1e-6, "Khz": 1e-3, "Mhz": 1.0, "Ghz": 1e3}.get(units[i], 1.0)
                d[f] = v
        d["dram_bytes_per_launch"] = d.get("dram_read_bytes", 0) + d.get("dram_write_bytes", 0)
        if d.get("lts_bytes"):
            d["lts_bytes_per_launch"] = d["lts_bytes"]
        if d.get("fma_cycles_active_sum") and d.get("fma_pipe_pct") and d.get("sm_cycles_active_sum"):
            d["fma_cycles_active_per_launch"] = d["fma_cycles_active_sum"]
            d["fma_cycles_per_sm_cycle"] = d["fma_cycles_active_sum"] / (
                d["fma_pipe_pct"] / 100.0 * d["sm_cycles_active_sum"])
        if d.get("l1_wavefronts_avg_per_sm") and d.get("l1_data_pipe_pct") and \
                d.get("sm_cycles_elapsed_avg"):
            # data-pipe wavefronts per launch (all SMs) and the per-SM-cycle peak
            d["l1_wavefronts_per_launch"] = 148 * d["l1_wavefronts_avg_per_sm"]
            d["l1_wavefronts_per_sm_cycle"] = d["l1_wavefronts_avg_per_sm"] / (
                d["l1_data_pipe_pct"] / 100.0 * d["sm_cycles_elapsed_avg"])
        if kind in res["kernels"] and res["kernels"][kind].get("duration_ms", 0) >= d.get(
                "duration_ms", 0):
            continue                      # keep the longest launch of a kind (full batch)
        res["kernels"][kind] = d
    Path(out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else sys.argv[1])

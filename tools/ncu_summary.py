"""Summarise an ncu --set full report into profiles/: the details page (CSV) and one traffic.json entry
(DRAM bytes per launch, duration, issue-slot use, pipes, shared-memory wavefronts and conflicts).
usage: python tools/ncu_summary.py REPORT.ncu-rep KEY KERNEL_LABEL SOURCE_NOTE DETAILS_CSV_OUT"""
import csv
import json
import os
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1,
         "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1, "s": 1e3}
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, key, label, note, details_out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    d = {}
    for k, un, x in zip(rows[0], rows[1], rows[2]):
        try:
            d[k] = (float(x.replace(",", "")), un)
        except ValueError:
            d[k] = (x, un)

    def val(k):
        return d[k][0] * SCALE.get(d[k][1], 1)

    def pct(k):
        return d[k][0] / 100 if k in d else None
    rec = {"kernel": label, "source": note,
           "bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
           "read": val("dram__bytes_read.sum"), "write": val("dram__bytes_write.sum"),
           "duration_ms": val("gpu__time_duration.sum"),
           "issue_slots_busy": pct("sm__inst_issued.avg.pct_of_peak_sustained_active"),
           "alu_pipe": pct("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
           "fma_pipe": pct("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
           # IMAD / IMAD.WIDE issue to the FMA-heavy half at half rate: the busier FMA half
           "fmaheavy_pipe": pct("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
           "warp_instructions_per_launch": d["smsp__inst_executed.sum"][0],
           "shared_wavefronts": d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"][0],
           "shared_bank_conflict_wavefronts": d["l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"][0],
           "l1_hit_rate": pct("l1tex__t_sector_hit_rate.pct"),
           "warps_active": pct("sm__warps_active.avg.pct_of_peak_sustained_active")}
    path = os.path.join(ROOT, "profiles", "r02", "traffic.json")
    t = json.load(open(path))
    t[key] = rec
    json.dump(t, open(path, "w"), indent=1)
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    open(details_out, "w").write(det)
    print(json.dumps({key: rec}))


if __name__ == "__main__":
    main(*sys.argv[1:6])

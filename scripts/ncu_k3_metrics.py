"""Extract the k_phase1 roofline inputs from an ncu --set full report.

    python scripts/ncu_k3_metrics.py <report.ncu-rep> <bench.log> <out.json>

The report must be the capture of the same bench command as <bench.log>
(whose JSON line carries the device counters of one query, incl. the
warp-record count of k_phase1 -- deterministic for the seeded workload).
bench.py reads <out.json> for the per-unit work and the DRAM traffic.
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "nsecond": 1e-6, "%": 1.0,
         "inst": 1.0, "": 1.0}


def main(rep, log, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:k_phase1"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = hdr.index(name)
        v = float(vals[i].replace(",", ""))
        return v * SCALE.get(units[i], 1.0)

    line = [x for x in open(log) if x.startswith("{")][-1]
    bench = json.loads(line)
    m = {
        "kernel": vals[hdr.index("Kernel Name")],
        "inst_executed": get("smsp__inst_executed.sum"),
        "warp_records": bench["counters"]["warp_records"],
        "dram_bytes": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
        "duration_ms_ncu": get("gpu__time_duration.sum"),
        "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fp64_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "fma_pct": get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "alu_pct": get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "source_report": rep,
    }
    m["inst_per_warp_record"] = m["inst_executed"] / m["warp_records"]
    with open(out, "w") as fh:
        json.dump(m, fh, indent=1)
    print(json.dumps(m, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])

"""DRAM traffic of one k_phase1 launch from an `ncu --page raw --csv` export:
    python scripts/ncu_traffic.py gpurun_out/ncu_full_raw.csv profiles/round2/k_phase1_traffic.json"""
import csv
import json
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
rows = list(csv.DictReader(open(sys.argv[1])))
units = rows[0]
for r in rows[1:]:
    if "k_phase1<double, 0, 0, 0>" in r["Kernel Name"].replace("(bool)", ""):
        rd = float(r["dram__bytes_read.sum"]) * UNIT[units["dram__bytes_read.sum"]]
        wr = float(r["dram__bytes_write.sum"]) * UNIT[units["dram__bytes_write.sum"]]
        out = {"kernel": r["Kernel Name"], "dram_read_bytes": rd, "dram_write_bytes": wr,
               "duration_ms_under_ncu": float(r["gpu__time_duration.sum"]) * {"ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3}.get(units["gpu__time_duration.sum"], 1),
               "source": "ncu --set full --clock-control none, one launch of the C5 bench step (profiles/round2/ncu_full_raw.csv)"}
        json.dump(out, open(sys.argv[2], "w"), indent=1)
        print(out)
        break
else:
    sys.exit("no k_phase1<double,0,0,0> launch in " + sys.argv[1])

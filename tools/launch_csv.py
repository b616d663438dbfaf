"""Condense an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv` launch list into one row per launch (reading aid for profiles/).

    python tools/launch_csv.py gpurun_out/launches.csv > profiles/rNN_launches.csv
"""
import csv
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
        "msecond": 1e6}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    launches = {}
    for r in rows:
        lid, name, metric, unit, val = r[0], r[4], r[12], r[13], r[14]
        d = launches.setdefault(int(lid), {"kernel": name[:60]})
        v = float(val.replace(",", "")) if val.replace(",", "").replace(".", "").isdigit() else None
        if v is not None:
            d[metric] = v * UNIT.get(unit, 1)
    w = csv.writer(sys.stdout)
    w.writerow(["id", "kernel", "gpu__time_duration_ns", "dram_read_bytes", "dram_write_bytes"])
    for lid in sorted(launches):
        d = launches[lid]
        w.writerow([lid, d["kernel"], int(d.get("gpu__time_duration.sum", 0)),
                    int(d.get("dram__bytes_read.sum", 0)), int(d.get("dram__bytes_write.sum", 0))])


if __name__ == "__main__":
    main(sys.argv[1])

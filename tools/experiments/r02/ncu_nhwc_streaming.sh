# ncu launch list (time, DRAM bytes) of one NHWC streaming forward + backward per shape
set -e
python tools/act_once.py leaky_relu NHWC 32x128x3136 bf16
for sh in ${SHAPES:-32x128x3136 32x1216x196}; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none ${NCU_EXTRA:-} --csv --log-file gpurun_out/ncu_$sh.csv python tools/act_once.py leaky_relu NHWC $sh bf16 > /dev/null 2>&1
done
python - <<'PY'
import csv, os
for sh in os.environ.get("SHAPES", "32x128x3136 32x1216x196").split():
    rows=list(csv.DictReader(l for l in open(f"gpurun_out/ncu_{sh}.csv") if l.startswith('"')))
    d={}
    for r in rows:
        d.setdefault((int(r["ID"]),r["Kernel Name"][:50]),{})[r["Metric Name"]]=r["Metric Value"]
    print(sh)
    for (i,k),v in sorted(d.items())[-6:]:
        print(" ",i,k,v.get("gpu__time_duration.sum"),v.get("dram__bytes_read.sum"),v.get("dram__bytes_write.sum"),v.get("lts__t_bytes.sum"))
PY

"""Convert an ncu --csv launch list (metrics dram__bytes_read.sum, dram__bytes_write.sum,
gpu__time_duration.sum) of the k_conv_tc launches of one config into
profiles/<round>/conv_dram_per_launch.csv, the per-launch DRAM traffic bench.py reports as
roofline.traffic.  Usage: python tools/conv_dram_csv.py ncu.csv out.csv"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
iid, ik, im, iu, iv = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1,
         "ms": 1e3, "msecond": 1e3}
launches = OrderedDict()
for r in data:
    if "k_conv_tc" not in r[ik]:
        continue
    d = launches.setdefault(r[iid], {"kernel": r[ik].split("(")[0]})
    d[r[im]] = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
with open(sys.argv[2], "w") as f:
    f.write("launch,kernel,dram_read_bytes,dram_write_bytes,duration_us\n")
    for i, d in enumerate(launches.values()):
        f.write(f"{i},{d['kernel']},{int(d.get('dram__bytes_read.sum', 0))},{int(d.get('dram__bytes_write.sum', 0))},"
                f"{d.get('gpu__time_duration.sum', 0):.2f}\n")
print(len(launches), "launches")

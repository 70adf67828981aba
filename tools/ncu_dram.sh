#!/bin/bash
# usage: ncu_dram.sh TAG [ENV=val ...]  -- per-kernel DRAM bytes / time of device-resident cfg4 reconstructions
# with caches left as the pipeline leaves them (--cache-control none), summed per kernel name over the capture.
tag=$1; shift
mkdir -p gpurun_out
env "$@" timeout 600 ncu --cache-control none --clock-control none --csv \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum \
  --log-file gpurun_out/dram_$tag.csv python tools/profile_step.py --iters 3 ${PROFILE_ARGS} > gpurun_out/dram_$tag.log 2>&1 || tail -3 gpurun_out/dram_$tag.log
python - gpurun_out/dram_$tag.csv "$tag" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[ix["Kernel Name"]].split("(")[0].split("::")[-1][:28]
    m, u, v = r[ix["Metric Name"]], r[ix["Metric Unit"]], float(r[ix["Metric Value"]].replace(",", ""))
    sc = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}.get(u, 1)
    a = agg.setdefault(name, collections.Counter()); a[m] += v * sc; a["n"] += 1
print("==", sys.argv[2])
for k, a in agg.items():
    n = a["n"] / 5
    print("%-28s n=%3d  rd %.3f GB  wr %.3f GB  t %.3f ms  l2 read hit %.2f" % (
        k, n, a["dram__bytes_read.sum"] / 1e9, a["dram__bytes_write.sum"] / 1e9, a["gpu__time_duration.sum"] * 1e3,
        a["lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum"] / max(1, a["lts__t_sectors_srcunit_tex_op_read.sum"])))
PY

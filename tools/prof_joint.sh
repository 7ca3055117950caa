#!/bin/bash
# per-kernel timing / pipe use of the joint-norm mode (config-2 shape)
python bench.py --score joint --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k 'regex:gram|apply|reduce|softmax' -s 30 -c 10 --csv --log-file gpurun_out/joint_k.csv \
    python bench.py --score joint --no-cpu-baseline --steps 2 --warmup 3 > /dev/null 2>&1
python tools/summarize_ncu.py metrics gpurun_out/joint_k.csv 2>/dev/null || python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/joint_k.csv")) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
for r in rows[1:]:
    print(r[ki][:48], r[mi], r[vi])
PY

for nc in 148 296 444 592 888; do
  TURBDA_JOINT_NCHUNK=$nc TURBDA_JOINT_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 30 --csv --log-file gpurun_out/nc$nc.csv python bench.py --config cfg2 --score joint --precision fp64 --steps 1 --warmup 3 --no-cpu-baseline --no-fp64 --no-e2e-variants > /dev/null 2>&1
  python tools/summarize_ncu.py launches gpurun_out/nc$nc.csv /tmp/nc.md > /dev/null; echo "nchunk $nc"; grep -E "gram|reduce" /tmp/nc.md
done

timeout 900 python -m pytest tests/test_gpu_determinism.py -q -p no:cacheprovider 2>&1 | tail -2
for env in "TURBDA_F32_FUSE_ALL=1" "TURBDA_F32_UNFUSED=1"; do
  env $env timeout 300 python tools/fused_breakdown.py 2097152 128
  env $env timeout 600 python tools/fused_breakdown.py 1048576 512
done
timeout 2400 bash tools/checked_run.sh

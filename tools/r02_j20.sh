bash tools/sweep_j20.sh "cfg1:0:0 cfg1:0:2 cfg1:0:3 cfg1:0:1 cfg1:2:2 cfg3:0:0 cfg3:1:2 cfg3:1:1 cfg3:2:2 cfg3:2:1 cfg3:1:3"
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "parity and not joint and not cycle" 2>&1 | tail -2
TURBDA_F32_J20=2 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "parity and not joint and not cycle" 2>&1 | tail -2

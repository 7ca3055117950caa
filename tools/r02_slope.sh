for spec in "8:0:0" "4:1:3" "4:1:0"; do
  IFS=: read wm fa j <<< "$spec"
  echo "== wmax:fuseall:j20 $spec"
  env TURBDA_F32_WMAX=$wm TURBDA_F32_FUSE_ALL=$fa TURBDA_F32_J20=$j timeout 200 python tools/steps_slope.py 8192 20
done
TURBDA_F32_UNFUSED=1 timeout 200 python tools/steps_slope.py 8192 20

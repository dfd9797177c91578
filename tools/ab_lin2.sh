# A/B of linearization variants (camera-major reduce blocks per SM / tile-pass blocks per SM)
VARS=${VARS:-"base cr2l2 cr3l2 cr3l3 cr4l2"}
for cfg in c5 c4; do for i in 1 2; do for v in $VARS; do
  POBA_LIB=libab/$v/libpoba.so python tools/time_lin.py $cfg 1.0 $v
done; done; done

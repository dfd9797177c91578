# A/B of the camera-major chunk size: bash tools/build_variant.sh c512 -DPOBA_CAM_CHUNK=512 (etc.) first
for i in 1 2; do for v in c512 c1024 c2048; do
  POBA_LIB=libab/$v/libpoba.so python tools/time_lin.py c5 1.0 $v
  POBA_LIB=libab/$v/libpoba.so python tools/time_lin.py c4 1.0 $v
done; done

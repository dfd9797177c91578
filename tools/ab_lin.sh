# A/B of linearize variants built by tools/build_variant.sh
# build the variants first, e.g. bash tools/build_variant.sh base; bash tools/build_variant.sh c512 -DPOBA_CAM_CHUNK=512
VARS=${VARS:?"set VARS to the libab/ variant names"}
for i in 1 2; do
for v in $VARS; do
  POBA_LIB=libab/$v/libpoba.so python tools/time_lin.py c5 1.0 $v
done; done

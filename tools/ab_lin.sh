# A/B of linearize variants built by tools/build_variant.sh
VARS=${VARS:-"ldcs ldg ldg64 ldg256"}
for i in 1 2; do
for v in $VARS; do
  POBA_LIB=libab/$v/libpoba.so python tools/time_lin.py c5 1.0 $v
done; done

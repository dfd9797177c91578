# A/B of term-kernel CTA shapes (warps per CTA x co-resident CTAs per SM); build first:
#   bash tools/build_variant.sh w6c2 "-DPOBA_TERM_WARPS=6 -DPOBA_TERM_CTAS=2"   etc.
VARS=${VARS:-"base w6c2 w4c3 w8c1"}
for i in 1 2; do for v in $VARS; do
  for cfg in c5 c4 c3; do POBA_LIB=libab/$v/libpoba.so python tools/time_term.py $cfg 1.0 $v; done
  POBA_LIB=libab/$v/libpoba.so python tools/time_term.py c5 1.0 $v 32
done; done

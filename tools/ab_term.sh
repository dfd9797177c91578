# A/B of term-kernel variants (build them first with tools/build_variant.sh): VARS="a b" bash tools/ab_term.sh
VARS=${VARS:?"set VARS to the libab/ variant names"}
for i in 1 2; do for v in $VARS; do
  POBA_LIB=libab/$v/libpoba.so python tools/time_term.py c5 1.0 $v
  POBA_LIB=libab/$v/libpoba.so python tools/time_term.py c4 1.0 $v
done; done

# A/B of term-kernel variants built by tools/build_variant.sh (see DESIGN.md / profiles)
VARS=${VARS:-"base rec16 perm perm64"}
for v in $VARS; do
  POBA_LIB=libab/$v/libpoba.so timeout 600 python -m pytest tests/test_gpu_scale_parity.py -q -x 2>&1 | tail -1 | sed "s/^/$v parity: /"
done
for i in 1 2; do
for v in $VARS; do
  POBA_LIB=libab/$v/libpoba.so python tools/time_term.py c5 1.0 $v
  POBA_LIB=libab/$v/libpoba.so python tools/time_term.py c4 1.0 $v
done; done

make -j16 >/dev/null 2>&1
for r in 0 1 2 3; do echo "rounds=$r"; POBA_LANE_ROUNDS=$r python tools/slot_stats.py c5:1.0 c4:1.0 2>&1 | grep stats; done
for i in 1 2; do for r in 0 2; do POBA_LANE_ROUNDS=$r python tools/time_term.py c5 1.0 rounds$r; POBA_LANE_ROUNDS=$r python tools/time_term.py c4 1.0 rounds$r; done; done 2>&1 | grep term
python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py tests/test_gpu_determinism.py -q -x 2>&1 | tail -2
python tools/det_op.py c3 0.1 300

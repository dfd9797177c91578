set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_prof.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_r01b.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/prof_term.py c5 1.0 > /dev/null 2>&1 || exit 2
ncu --set full --clock-control none --import-source on -k regex:k_term -s 2 -c 1 -o gpurun_out/term_c5_full_r01b python tools/prof_term.py c5 1.0 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log

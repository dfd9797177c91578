# one gpurun call: bench line, launch list, ncu --set full of the term kernel (C5)
# usage (under gpurun): bash tools/prof_cmd.sh TAG
TAG=${1:-r01}
set -x
python bench.py > gpurun_out/bench_${TAG}.log 2>&1 || exit 1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_prof_${TAG}.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c5_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${TAG}.log 2>&1
python tools/prof_term.py c5 1.0 > /dev/null 2>&1 || exit 2
ncu --set full --clock-control none --import-source on -k regex:k_term -s 2 -c 1 -o gpurun_out/term_c5_full_${TAG} python tools/prof_term.py c5 1.0 > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
tail -1 gpurun_out/bench_${TAG}.log

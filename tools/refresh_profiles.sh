#!/bin/bash
# Runs ON the GPU box (via gpurun): full GPU test suite, the default bench line, the ncu launch
# list of a short bench run, and one `ncu --set full` capture per hot kernel.  Outputs land in
# gpurun_out/ (scratch); tools/ncu_summary.py turns the captures into profiles/ncu_summary.json.
TAG=${1:-r02}
O=gpurun_out
timeout -s KILL 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.txt 2>&1
tail -3 $O/pytest_gpu_$TAG.txt
python bench.py > $O/bench_full_$TAG.json 2> $O/bench_full_$TAG.err
tail -c 600 $O/bench_full_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_bench_$TAG.json 2>&1
NCU="ncu --set full --clock-control none --import-source on -c 1"
$NCU -k regex:'decode_kernel' -s 3 -o $O/prof_dec_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1
$NCU -k regex:'train_kernel' -s 3 -o $O/prof_tr_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras > /dev/null 2>&1
# the three full captures together can exceed gpurun's 64 MiB copy-back: MULTI=only / MULTI=skip
[ "${MULTI:-}" != skip ] && $NCU -k regex:'decode_multi_kernel' -s 1 -o $O/prof_multi_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls $O | grep $TAG

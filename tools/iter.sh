#!/bin/bash
# usage: tools/iter.sh TAG [pytest-args]   -- GPU tests + bench + ncu full capture of decode_kernel
TAG=$1; shift
T=${TESTS:-tests/test_gpu_decode.py}
/usr/local/graft/bin/gpurun --timeout 1200 -- "timeout -s KILL 600 python -m pytest $T -x -q $* 2>&1 | tail -15; python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-decode_kernel} -s ${KSKIP:-3} -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log" 2>&1 | grep -v "^\[gpurun\] sending" | tail -12
python - <<PY
import json
try:
    d=json.load(open('gpurun_out/bench_$TAG.json'))
    print('value', round(d['value'],3), 'ms/step', round(d['ms_per_step'],4), 'frac', d['roofline']['frac'], 'clk', d['clocks'].get('sm_mhz'), 'train', d.get('train',{}).get('value'))
except Exception as e:
    print('bench parse failed', e); print(open('gpurun_out/bench_$TAG.err').read()[-2000:])
PY
if [ -f gpurun_out/prof_$TAG.ncu-rep ]; then
  ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass 2>/dev/null > /tmp/sass_$TAG.csv
  ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv 2>/dev/null > /tmp/raw_$TAG.csv
  python tools/sass_profile.py /tmp/sass_$TAG.csv 0 | head -25
  python tools/raw_summary.py /tmp/raw_$TAG.csv
fi

#!/bin/bash
# Round-2b final refresh: full GPU suite, smoke, a bench line per config
# (timed regions >= ~1 s, CPU baseline on), the launch list of the default
# command and an ncu capture of the C3 kernel.  Outputs under gpurun_out/r2b/.
O=gpurun_out/r2b
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench_C3.json 2> $O/bench_C3.err
for cs in ${CFGS:-C1:300 C2:50 C4:250 C4b:200 C5:20 C3LM:4}; do
  c=${cs%%:*}; k=${cs##*:}
  timeout 1200 python bench.py --config $c --steps $k --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
  --log-file $O/launches_C3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain6_step -s 1 -c 1 \
  -o $O/ncu_C3 -f python scripts/prof_run.py C3 4096 2 > $O/ncu_C3.log 2>&1
tail -n 3 $O/pytest_gpu.log; tail -n 2 $O/smoke.log
for f in $O/bench_*.json; do echo $f $(tail -n 1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], round(d['value']), d['roofline']['frac'], d['e2e']['value'], (d['cpu_baseline'] or {}).get('value'), d['gpu_launches'])" 2>&1 | tail -n 1); done

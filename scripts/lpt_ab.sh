#!/bin/bash
# LPT launch order A/B (tree / residual kernels) + parity.  gpurun_out/lpt/
O=gpurun_out/lpt; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_tree.py tests/test_gpu_resid.py tests/test_gpu_energy_lm.py tests/test_gpu_fullsize.py -q -x > $O/parity.log 2>&1; echo "rc $?" >> $O/parity.log
for c in C4:50 C4b:50 C3LM:3 C5:2; do
  cfg=${c%%:*}; k=${c##*:}
  timeout 900 python bench.py --config $cfg --steps $k --warmup 3 --no-cpu-baseline > $O/on_$cfg.json 2>/dev/null
  PBAD_GPU_NO_LPT=1 timeout 900 python bench.py --config $cfg --steps $k --warmup 3 --no-cpu-baseline > $O/off_$cfg.json 2>/dev/null
done
tail -n 2 $O/parity.log
for f in $O/on_*.json $O/off_*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['mean_iterations_per_step'])"); done

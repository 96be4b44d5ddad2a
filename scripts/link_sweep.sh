#!/bin/bash
# The metric's "vs N links": C3's chain scene (make_chain_scene(N/2): N/2 massless Z-hinges +
# N/2 Y-hinge boxes), L-BFGS, dt = 0.1, batch 4096, at N links.  gpurun_out/sweep/
O=gpurun_out/sweep; mkdir -p $O
for N in 20 50 100 200 300; do
  timeout 900 python bench.py --config C3 --links $N --steps 3 --warmup 3 --no-cpu-baseline > $O/C3_N$N.json 2> $O/C3_N$N.err
done
for N in 10 25 50 100; do
  timeout 900 python bench.py --config C2 --links $N --steps 10 --warmup 3 --no-cpu-baseline > $O/C2_N$N.json 2> $O/C2_N$N.err
done
for f in $O/*.json; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], round(d['value']), round(d['roofline']['frac'],4), d['kernel'][:22], d['mean_iterations_per_step'])" 2>&1 | tail -1); done

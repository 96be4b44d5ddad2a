for b in 1024 2048 3072 4096 6144 8192; do
  PBAD_BENCH_BATCH=$b timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($b, d['ms_per_step'], d['value'])"
done

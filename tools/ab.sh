# A/B timing of libraries on one box: bash tools/ab.sh libA.so libB.so [libC.so ...]
# (extra bench args via BENCH_ARGS).  Two rounds over the list; prints ms_per_step per run.
for r in 1 2; do
  for L in "$@"; do
    printf "%s " $L
    DILU_LIB=paper_2503_05130_b200/$L python bench.py --no-cpu-baseline --e2e-steps 0 --no-secondary --steps 3 $BENCH_ARGS | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'])"
  done
done

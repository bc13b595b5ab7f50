# A/B timing of side libraries on one box: bash tools/ab.sh libA.so libB.so [extra bench args]
# Alternates A, B, A, B and prints ms_per_step of each run.
A=$1; B=$2; shift 2
for r in 1 2; do
  for L in $A $B; do
    printf "%s " $L
    DILU_LIB=paper_2503_05130_b200/$L python bench.py --no-cpu-baseline --e2e-steps 0 "$@" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'])"
  done
done

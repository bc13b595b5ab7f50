D=gpurun_out/r2r
mkdir -p $D
for L in libdilu_mc.so libdilu_r72.so libdilu_r64.so; do
  for T in auto 160 192; do
    printf "$L $T " >> $D/ab.txt
    if [ $T = auto ]; then unset DILU_THREADS; else export DILU_THREADS=$T; fi
    DILU_VERBOSE=1 DILU_LIB=paper_2503_05130_b200/$L python bench.py --no-cpu-baseline --e2e-steps 0 --no-secondary --steps 2 2> $D/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'])" >> $D/ab.txt 2>&1
    grep "cta engine" $D/err.txt >> $D/ab.txt
  done
done
unset DILU_THREADS
for SC in 8 1; do
  DILU_VERBOSE=1 timeout 600 python bench.py --workload C5 --scenarios $SC --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/bench_c5_s$SC.json 2> $D/bench_c5_s$SC.err
done
DILU_VERBOSE=1 DILU_GROUP=10 DILU_CLUSTER=10 timeout 600 python bench.py --workload C5 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/bench_c5_k10.json 2> $D/bench_c5_k10.err
timeout 1500 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu.txt
ls -la $D

D=gpurun_out/r2s
mkdir -p $D
bash tools/ab.sh libdilu_prev.so libdilu.so > $D/ab.txt 2>&1
for SC in 8 1; do
  DILU_VERBOSE=1 timeout 300 python bench.py --workload C5 --scenarios $SC --slots 3600 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/bench_c5_s$SC.json 2> $D/bench_c5_s$SC.err; echo "rc $?" >> $D/bench_c5_s$SC.err
done
DILU_VERBOSE=1 DILU_GROUP=10 DILU_CLUSTER=10 timeout 300 python bench.py --workload C5 --slots 3600 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/bench_c5_k10.json 2> $D/bench_c5_k10.err
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "multicluster" > $D/pytest_mc.txt 2>&1; echo "rc $?" >> $D/pytest_mc.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu.txt
ls -la $D

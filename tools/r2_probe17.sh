D=gpurun_out/r2q
mkdir -p $D
bash tools/ab.sh libdilu_prev.so libdilu_rcpdiv.so > $D/ab.txt 2>&1
DILU_LIB=paper_2503_05130_b200/libdilu_prev_timing.so timeout 300 python tools/c4_phase_breakdown.py > $D/phase_c4.json 2>&1
DILU_LIB=paper_2503_05130_b200/libdilu_prev.so timeout 600 python bench.py --workload C5 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/bench_c5.json 2> $D/bench_c5.err
ls -la $D

# Round-2 final evidence on the GPU box (final build): parity suite (normal and bounds-checked
# library), smoke, bench lines, ncu launch list and full captures, phase breakdowns.
# Run: gpurun -- bash tools/collect_r2.sh   (compute-sanitizer is closed on this pool)
set -x
D=gpurun_out/r2final
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > $D/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $D/pytest_gpu.txt 2>&1; echo "rc $?" >> $D/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; echo "rc $?" >> $D/smoke.txt
python bench.py > $D/bench_c4.json 2> $D/bench_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > $D/ref_c4.json 2>&1
DILU_VERBOSE=1 python bench.py --workload C5 --steps 3 --warmup 1 > $D/bench_c5.json 2> $D/bench_c5.err
DILU_VERBOSE=1 python bench.py --workload C5 --scenarios 1 --steps 3 --warmup 1 --no-cpu-baseline > $D/bench_c5_s1.json 2> $D/bench_c5_s1.err
python bench.py --vertical alg2 --steps 3 --warmup 3 > $D/bench_c4_alg2.json 2> $D/bench_c4_alg2.err
python bench.py --latency --steps 3 --warmup 3 > $D/bench_c4_latency.json 2> $D/bench_c4_latency.err
python bench.py --workload PROFILE > $D/bench_profile.json 2> $D/bench_profile.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > $D/bench_c4_torchrun.json 2> $D/bench_c4_torchrun.err
python bench.py --gpus 2 > $D/bench_gpus2_refusal.txt 2>&1; echo "rc $?" >> $D/bench_gpus2_refusal.txt
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_runILb1ELi0 -s 1 -c 1 -o $D/c4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_run_clusterILi1 -s 1 -c 1 -o $D/c5_full python bench.py --workload C5 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/ncu_c5.log 2>&1
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so timeout 600 python tools/c4_phase_breakdown.py > $D/phase_c4.json 2> $D/phase_c4.err
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so timeout 900 python tools/c5_phase_breakdown.py > $D/phase_c5.json 2> $D/phase_c5.err
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so timeout 900 python tools/c5_phase_breakdown.py 1200 burst > $D/phase_c5_burst.json 2> $D/phase_c5_burst.err
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_bounds.so timeout 1800 python -m pytest tests -m gpu -q > $D/pytest_gpu_bounds.txt 2>&1; echo "rc $?" >> $D/pytest_gpu_bounds.txt
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_bounds.so timeout 900 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/bench_bounds.json 2> $D/bench_bounds.err
ls -la $D

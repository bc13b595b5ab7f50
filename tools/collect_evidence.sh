# Round-1 evidence: bench lines (C4, C5, C4 Alg.2, C4 latency, profiler, oracle arm), the
# ncu launch list of the default bench command and ncu --set full captures of the C4 and
# C5 kernels, all under gpurun_out/r1f/.
# Run on the GPU box: gpurun -- bash tools/collect_evidence.sh
set -x
D=gpurun_out/r1i
mkdir -p $D
python bench.py > $D/bench_c4.json 2> $D/bench_c4.err
python bench.py --workload C5 > $D/bench_c5.json 2> $D/bench_c5.err
python bench.py --vertical alg2 --steps 3 --warmup 3 > $D/bench_c4_alg2.json 2> $D/bench_c4_alg2.err
python bench.py --latency --steps 3 --warmup 3 > $D/bench_c4_latency.json 2> $D/bench_c4_latency.err
python bench.py --workload PROFILE > $D/bench_profile.json 2> $D/bench_profile.err
python bench.py --impl reference --steps 2 --warmup 1 > $D/ref_c4.json 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > $D/bench_c4_torchrun.json 2> $D/bench_c4_torchrun.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_runILb1ELi0 -s 1 -c 1 -o $D/c4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $D/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_run_clusterILi1 -c 1 -o $D/c5_full python bench.py --workload C5 --slots 3600 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > $D/ncu_c5.log 2>&1
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so python tools/c4_phase_breakdown.py > $D/phase_c4.json 2>&1
ls -la $D

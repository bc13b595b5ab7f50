# Round-1 evidence: bench lines (C4, C5, C4 Alg.2, oracle arm), the ncu launch list and
# ncu --set full captures of the C4 and C5 kernels, all under gpurun_out/r1b/.
# Run on the GPU box: gpurun -- bash tools/collect_evidence.sh
set -x
mkdir -p gpurun_out/r1b
python bench.py > gpurun_out/r1b/bench_c4.json 2> gpurun_out/r1b/bench_c4.err
python bench.py --workload C5 > gpurun_out/r1b/bench_c5.json 2> gpurun_out/r1b/bench_c5.err
python bench.py --vertical alg2 --steps 3 --warmup 3 > gpurun_out/r1b/bench_c4_alg2.json 2> gpurun_out/r1b/bench_c4_alg2.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1b/ref_c4.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1b/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_runILb1ELi0 -s 1 -c 1 -o gpurun_out/r1b/c4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r1b/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_run_clusterILi1 -c 1 -o gpurun_out/r1b/c5_full python bench.py --workload C5 --slots 3600 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r1b/ncu_c5.log 2>&1
ls -la gpurun_out/r1b

# Round-2 evidence on the GPU box (final build): bench lines, ncu launch list and full
# captures, sanitizers, modes report.  Run: gpurun -- bash tools/collect_r2.sh
set -x
D=gpurun_out/r2final
mkdir -p $D
python bench.py > $D/bench_c4.json 2> $D/bench_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > $D/ref_c4.json 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > $D/bench_c4_torchrun.json 2> $D/bench_c4_torchrun.err
python bench.py --gpus 2 > $D/bench_gpus2_refusal.txt 2>&1; echo "rc $?" >> $D/bench_gpus2_refusal.txt
DILU_VERBOSE=1 python bench.py --workload C5 --steps 3 --warmup 1 > $D/bench_c5.json 2> $D/bench_c5.err
DILU_VERBOSE=1 python bench.py --workload C5 --scenarios 1 --steps 3 --warmup 1 --no-cpu-baseline > $D/bench_c5_s1.json 2> $D/bench_c5_s1.err
python bench.py --vertical alg2 --steps 3 --warmup 3 > $D/bench_c4_alg2.json 2> $D/bench_c4_alg2.err
python bench.py --latency --steps 3 --warmup 3 > $D/bench_c4_latency.json 2> $D/bench_c4_latency.err
python bench.py --workload PROFILE > $D/bench_profile.json 2> $D/bench_profile.err
python tools/modes_report.py --out $D/modes_report.json > /dev/null 2> $D/modes_report.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $D/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_runILb1ELi0 -s 1 -c 1 -o $D/c4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/ncu_c4.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_run_clusterILi1 -c 1 -o $D/c5_full python bench.py --workload C5 --slots 3600 --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/ncu_c5.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck initcheck; do
  for W in "c2 --slots 900" "c4slice --slots 300 --every 455" "c5win --slots 100"; do
    echo "== $T $W" >> $D/sanitizer.txt
    timeout 900 $CS --tool $T --print-limit 10 python tools/san_run.py $W 2>&1 | grep -E "ERROR SUMMARY|PASS|FAIL|Error" >> $D/sanitizer.txt
  done
done
for O in 0 1; do
  echo "== racecheck c4slice DILU_NO_OVL=$O" >> $D/sanitizer.txt
  DILU_NO_OVL=$O timeout 1200 $CS --tool racecheck --racecheck-report analysis --print-limit 10 python tools/san_run.py c4slice --slots 60 --every 1024 2>&1 | grep -E "RACECHECK SUMMARY|PASS|FAIL" >> $D/sanitizer.txt
done
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_bounds.so timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/bench_bounds.json 2> $D/bench_bounds.err
ls -la $D

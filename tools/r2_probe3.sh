# Round-2 third GPU call: term_smem probe, phase breakdown, ncu source capture, pad sweep.
D=gpurun_out/r2c
mkdir -p $D
L=paper_2503_05130_b200
DILU_LIB=$L/libdilu_dilu_term_smem_dilu_term_probe.so timeout 300 python tools/san_run.py c2 > $D/term_probe_c2.txt 2>&1; echo "rc $?" >> $D/term_probe_c2.txt
timeout 600 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu.txt
timeout 300 python bench.py --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err
DILU_LIB=$L/libdilu_dilu_phase_timing.so timeout 300 python tools/c4_phase_breakdown.py > $D/phase_c4.json 2>&1
for P in 1024 4096; do
  for W in "c2" "c4slice --every 7 --slots 3600"; do
    echo "== pad $P $W" >> $D/pad.txt
    DILU_LIB=$L/libdilu_dilu_hot_pad_$P.so timeout 300 python tools/san_run.py $W >> $D/pad.txt 2>&1; echo "rc $?" >> $D/pad.txt
  done
done
DILU_LIB=$L/libdilu_dilu_hot_pad_1024.so timeout 240 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $D/bench_pad1024.json 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_runILb1ELi0 -s 1 -c 1 -o $D/c4_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $D/ncu_full.log 2>&1
ls -la $D

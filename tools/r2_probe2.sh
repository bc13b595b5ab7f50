# Round-2 second GPU call: bounds-checked library over every parity case, padded layout at
# full C4 size, terminate in shared space under memcheck.
D=gpurun_out/r2b
mkdir -p $D
B=paper_2503_05130_b200/libdilu_dilu_bounds.so
BP=paper_2503_05130_b200/libdilu_dilu_bounds_dilu_hot_pad.so
for W in "c2 --seed 0" "c2 --seed 1" "c2 --seed 2" "c4slice" "c4slice --every 7 --slots 3600" "c1" "c5win --slots 600" "c3win --slots 600"; do
  echo "== bounds $W" >> $D/bounds.txt
  DILU_LIB=$B timeout 300 python tools/san_run.py $W >> $D/bounds.txt 2>&1; echo "rc $?" >> $D/bounds.txt
done
for W in "c2 --seed 0" "c4slice --every 7 --slots 3600"; do
  echo "== bounds+pad $W" >> $D/bounds.txt
  DILU_LIB=$BP timeout 300 python tools/san_run.py $W >> $D/bounds.txt 2>&1; echo "rc $?" >> $D/bounds.txt
done
DILU_LIB=$B timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > $D/bench_bounds.json 2> $D/bench_bounds.err; echo "rc $?" >> $D/bench_bounds.err
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_hot_pad.so timeout 240 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 > $D/bench_pad.json 2> $D/bench_pad.err; echo "rc $?" >> $D/bench_pad.err
DILU_LIB=$BP timeout 600 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0 > $D/bench_bounds_pad.json 2> $D/bench_bounds_pad.err; echo "rc $?" >> $D/bench_bounds_pad.err
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_term_smem.so timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --print-limit 20 python tools/san_run.py c2 > $D/san_memcheck_c2full_termsmem.txt 2>&1; echo "rc $?" >> $D/san_memcheck_c2full_termsmem.txt
DILU_LIB=$B timeout 1500 python -m pytest tests -m gpu -x -q > $D/pytest_gpu_bounds.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu_bounds.txt
ls -la $D

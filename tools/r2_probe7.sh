D=gpurun_out/r2g
mkdir -p $D
bash tools/ab.sh libdilu_base_r2a.so libdilu.so libdilu_dilu_view_copy.so > $D/ab.txt 2>&1
for T in 128 160 192 224; do
  printf "threads $T " >> $D/threads.txt
  DILU_THREADS=$T DILU_LIB=paper_2503_05130_b200/libdilu_base_r2a.so python bench.py --no-cpu-baseline --e2e-steps 0 --no-secondary --steps 2 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'])" >> $D/threads.txt 2>&1
done
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so timeout 300 python tools/c4_phase_breakdown.py > $D/phase_c4.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "launch_shape or c2_full or c1" > $D/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu.txt
ls -la $D

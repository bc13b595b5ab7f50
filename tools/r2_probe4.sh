D=gpurun_out/r2d
mkdir -p $D
timeout 900 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu.txt
bash tools/ab.sh libdilu_base_r2a.so libdilu.so > $D/ab.txt 2>&1
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_bounds.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c2 or c4 or place or cold or shard or c1" > $D/pytest_bounds.txt 2>&1; echo "rc $?" >> $D/pytest_bounds.txt
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so timeout 300 python tools/c4_phase_breakdown.py > $D/phase_c4.json 2>&1
timeout 600 python bench.py > $D/bench_c4.json 2> $D/bench_c4.err
ls -la $D

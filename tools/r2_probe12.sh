D=gpurun_out/r2l
mkdir -p $D
timeout 900 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu.txt
DILU_THREADS=256 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c2_full or c4_sample or launch" > $D/pytest_gpu_t256.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu_t256.txt
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_bounds.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c2 or c4 or place or cold or shard or c1 or split or launch" > $D/pytest_bounds.txt 2>&1; echo "rc $?" >> $D/pytest_bounds.txt
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so timeout 300 python tools/c4_phase_breakdown.py > $D/phase_c4.json 2>&1
DILU_THREADS=256 DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so timeout 300 python tools/c4_phase_breakdown.py > $D/phase_c4_t256.json 2>&1
ls -la $D

D=gpurun_out/r2p
mkdir -p $D
bash tools/ab.sh libdilu_prev.so libdilu_b1warp.so libdilu_b1div.so > $D/ab.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu.txt
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_bounds.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c2 or c4 or place or cold or shard or c1 or split or launch or c5_shaped or fused" > $D/pytest_bounds.txt 2>&1; echo "rc $?" >> $D/pytest_bounds.txt
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so timeout 300 python tools/c4_phase_breakdown.py > $D/phase_c4.json 2>&1
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool initcheck --print-limit 20 python tools/san_run.py c2 --slots 900 > $D/san_initcheck_c2.txt 2>&1; echo "rc $?" >> $D/san_initcheck_c2.txt
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool initcheck --print-limit 20 python tools/san_run.py c4slice --slots 300 --every 455 > $D/san_initcheck_c4.txt 2>&1; echo "rc $?" >> $D/san_initcheck_c4.txt
ls -la $D

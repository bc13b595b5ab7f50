D=gpurun_out/r2o
mkdir -p $D
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_phase_timing.so timeout 300 python tools/c5_phase_breakdown.py 3600 > $D/phase_c5.json 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck initcheck; do
  timeout 900 $CS --tool $T --print-limit 20 python tools/san_run.py c2 --slots 900 > $D/san_${T}_c2.txt 2>&1; echo "rc $?" >> $D/san_${T}_c2.txt
  timeout 900 $CS --tool $T --print-limit 20 python tools/san_run.py c4slice --slots 300 --every 455 > $D/san_${T}_c4.txt 2>&1; echo "rc $?" >> $D/san_${T}_c4.txt
done
timeout 1200 $CS --tool racecheck --racecheck-report analysis --print-limit 20 python tools/san_run.py c4slice --slots 60 --every 1024 > $D/san_racecheck_c4_ovl.txt 2>&1; echo "rc $?" >> $D/san_racecheck_c4_ovl.txt
DILU_NO_OVL=1 timeout 1200 $CS --tool racecheck --racecheck-report analysis --print-limit 20 python tools/san_run.py c4slice --slots 60 --every 1024 > $D/san_racecheck_c4_noovl.txt 2>&1; echo "rc $?" >> $D/san_racecheck_c4_noovl.txt
timeout 900 $CS --tool memcheck --print-limit 20 python tools/san_run.py c5win --slots 100 > $D/san_memcheck_c5.txt 2>&1; echo "rc $?" >> $D/san_memcheck_c5.txt
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_vmode_2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c2_full or c4 or c1 or place or launch" > $D/pytest_vmode2.txt 2>&1; echo "rc $?" >> $D/pytest_vmode2.txt
ls -la $D

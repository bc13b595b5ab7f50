D=gpurun_out/r2n
mkdir -p $D
for L in libdilu_base_r2a.so libdilu.so libdilu_dilu_vmode_2.so; do
  for T in auto 256; do
    printf "$L $T " >> $D/ab.txt
    if [ $T = auto ]; then unset DILU_THREADS; else export DILU_THREADS=$T; fi
    DILU_LIB=paper_2503_05130_b200/$L python bench.py --no-cpu-baseline --e2e-steps 0 --no-secondary --steps 2 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'])" >> $D/ab.txt 2>&1
  done
done
unset DILU_THREADS
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_runILb1ELi0 -s 1 -c 1 -o $D/c4 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/ncu.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu.txt
ls -la $D

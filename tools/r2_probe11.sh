D=gpurun_out/r2k
mkdir -p $D
for L in libdilu_base_r2a.so libdilu.so libdilu_dilu_vmode_1.so libdilu_dilu_vmode_2.so; do
  for T in auto 160 256; do
    printf "$L $T " >> $D/ab.txt
    if [ $T = auto ]; then unset DILU_THREADS; else export DILU_THREADS=$T; fi
    DILU_VERBOSE=1 DILU_LIB=paper_2503_05130_b200/$L python bench.py --no-cpu-baseline --e2e-steps 0 --no-secondary --steps 2 2>$D/err_$L_$T.txt | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'])" >> $D/ab.txt 2>&1
    grep "cta engine" $D/err_$L_$T.txt >> $D/ab.txt
  done
done
unset DILU_THREADS
ls -la $D

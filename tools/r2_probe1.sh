# Round-2 first GPU call: regression tests, baseline bench, layout variants, sanitizers.
D=gpurun_out/r2a
mkdir -p $D
nvidia-smi > $D/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $D/pytest_gpu.txt 2>&1; echo "pytest rc $?" >> $D/pytest_gpu.txt
timeout 300 python bench.py --no-cpu-baseline > $D/bench_c4.json 2> $D/bench_c4.err
for L in libdilu_dilu_hot_pad.so libdilu_dilu_term_smem.so; do
  for W in c2 c4slice; do
    echo "== $L $W" >> $D/variants.txt
    DILU_LIB=paper_2503_05130_b200/$L timeout 120 python tools/san_run.py $W >> $D/variants.txt 2>&1; echo "rc $?" >> $D/variants.txt
  done
done
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck initcheck; do
  timeout 600 $CS --tool $T --print-limit 50 python tools/san_run.py c2 --slots 600 > $D/san_${T}_c2.txt 2>&1; echo "rc $?" >> $D/san_${T}_c2.txt
  timeout 600 $CS --tool $T --print-limit 50 python tools/san_run.py c4slice --slots 300 --every 455 > $D/san_${T}_c4.txt 2>&1; echo "rc $?" >> $D/san_${T}_c4.txt
done
DILU_NO_OVL=1 timeout 600 $CS --tool memcheck --print-limit 50 python tools/san_run.py c4slice --slots 300 --every 455 > $D/san_memcheck_c4_noovl.txt 2>&1; echo "rc $?" >> $D/san_memcheck_c4_noovl.txt
DILU_LIB=paper_2503_05130_b200/libdilu_dilu_term_smem.so timeout 600 $CS --tool memcheck --print-limit 50 python tools/san_run.py c2 --slots 600 > $D/san_memcheck_c2_termsmem.txt 2>&1; echo "rc $?" >> $D/san_memcheck_c2_termsmem.txt
ls -la $D

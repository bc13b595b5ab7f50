D=gpurun_out/r2j
mkdir -p $D
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_runILb1ELi0 -s 1 -c 1 -o $D/c4_narrow python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/ncu_narrow.log 2>&1
DILU_LIB=paper_2503_05130_b200/libdilu_base_r2a.so ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_runILb1ELi0 -s 1 -c 1 -o $D/c4_base python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/ncu_base.log 2>&1
ls -la $D

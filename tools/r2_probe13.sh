D=gpurun_out/r2m
mkdir -p $D
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_runILb1ELi0 -s 1 -c 1 -o $D/c4_m1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary > $D/ncu_m1.log 2>&1
python tools/modes_report.py > $D/modes_report.json 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_profile.py -x -q -k "modes_directional or load" > $D/pytest_new.txt 2>&1; echo "rc $?" >> $D/pytest_new.txt
ls -la $D

D=gpurun_out/r2t
mkdir -p $D
run() { # scenarios group cluster
  printf "S=$1 K=$2 Kc=$3 " >> $D/c5_shapes.txt
  DILU_GROUP=$2 DILU_CLUSTER=$3 DILU_VERBOSE=1 timeout 300 python bench.py --workload C5 --scenarios $1 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-secondary 2> $D/err.txt | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'])" >> $D/c5_shapes.txt 2>&1
  grep "cluster engine" $D/err.txt >> $D/c5_shapes.txt
}
run 8 10 10
run 8 12 6
run 8 16 8
run 8 18 9
run 8 18 2
run 1 16 16
run 1 32 16
run 1 64 16
run 1 144 12
run 1 148 4
ls -la $D

# one ncu --set full capture of gp_tc_kernel for a bench config under extra env: tools/gpu_ncu_env.sh CONFIG OUT VAR=VAL...
cfg=$1; out=$2; shift 2
CMD="python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu"
env "$@" $CMD > gpurun_out/plain_$out.log 2>&1 && \
env "$@" ncu --set full --clock-control none --import-source on -k regex:"gp_tc_kernel" -s 1 -c 1 -o gpurun_out/$out $CMD > gpurun_out/ncu_$out.log 2>&1
echo ncu=$?

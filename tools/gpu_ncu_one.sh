# one ncu --set full capture of a kernel of one bench config: tools/gpu_ncu_one.sh CONFIG REGEX OUT
CMD="python bench.py --config $1 --steps 2 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain_$3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$2" -s 1 -c 1 -o gpurun_out/$3 $CMD > gpurun_out/ncu_$3.log 2>&1
echo ncu=$?

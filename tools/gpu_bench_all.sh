# round-2 measurement set (one gpurun call): both bench arms on the default config, the other
# configs, the launch list and one ncu --set full capture of the step kernels (M200)
set -x
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" > gpurun_out/host_cpu.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv >> gpurun_out/host_cpu.txt
python bench.py --impl reference > gpurun_out/bench_ref_M200.json 2> gpurun_out/bench_ref_M200.err
python bench.py > gpurun_out/bench_M200_full.json 2> gpurun_out/bench_M200_full.err
python bench.py --config C3 --no-cpu > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
python bench.py --config C5 --no-cpu --steps 20 > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
CMD="python bench.py --config M200 --steps 2 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_M200.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gp_tc_kernel|rf_qs_summary|merge" -s 3 -c 3 -o gpurun_out/prof_M200_final $CMD > gpurun_out/ncu2.log 2>&1
echo ncu=$?

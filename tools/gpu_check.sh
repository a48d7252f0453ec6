set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
for c in M200 C3 C5; do BX_QS_INFO=1 python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
CMD="python bench.py --config M200 --steps 2 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_M200.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gp_tc_kernel|rf_qs_summary" -s 2 -c 2 -o gpurun_out/prof_M200 $CMD > gpurun_out/ncu2.log 2>&1
echo ncu=$?
tail -3 gpurun_out/gpu_tests.log

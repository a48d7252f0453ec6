timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final2_gpu_tests.log 2>&1; echo tests=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2_smoke.log 2>&1; echo smoke=$?
python bench.py > gpurun_out/final2_bench.json 2> gpurun_out/final2_bench.err; echo bench=$?
python bench.py --impl reference > gpurun_out/final2_bench_ref.json 2> gpurun_out/final2_bench_ref.err; echo ref=$?
for c in C3 C5; do python bench.py --config $c --no-cpu > gpurun_out/final2_bench_$c.json 2> gpurun_out/final2_bench_$c.err; done
CMD="python bench.py --config M200 --steps 2 --warmup 1 --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final2_launches_M200.csv $CMD > gpurun_out/final2_ncu1.log 2>&1; echo ncu=$?

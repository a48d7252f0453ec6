# zero-copy posterior: kernel durations with the separate packed buffer (0), without it (32), and
# over a device copy of the pool (128)
for d in 0 32 128; do
BX_TC_DEBUG=$d ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e2e_dbg$d.csv python tools/e2e_gap.py 2 > gpurun_out/e2e_dbg$d.log 2>&1
done

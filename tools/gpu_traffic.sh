# single-pass DRAM traffic of the step kernels (M200, C3) and one --set full capture (M200 step)
for c in M200 C3; do
  python tools/profile_run.py $c 2 > gpurun_out/plain_$c.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:"gp_tc_kernel|rf_qs_summary|merge_fast" --csv --log-file gpurun_out/traffic_$c.csv \
      python tools/profile_run.py $c 2 > gpurun_out/ncu_t_$c.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"gp_tc_kernel|rf_qs_summary" -s 2 -c 2 \
    -o gpurun_out/prof_M200_step python tools/profile_run.py M200 2 > gpurun_out/ncu_full.log 2>&1
echo ncu=$?

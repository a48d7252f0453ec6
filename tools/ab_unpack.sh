# timing experiment: the zero-copy posterior with and without the decoders' write-back of the
# unpacked rows (ab_v built by tools/build_variant.sh; its results are wrong, only the time counts)
for side in . ab_v; do
  (cd $side && BX_TC_DEBUG=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OLDPWD/gpurun_out/unpack_$(basename $side).csv python tools/e2e_gap.py 2 > /dev/null 2>&1)
done

for i in 1 2 3; do
  for side in ab_old .; do
    echo "== $side"; (cd $side && python tools/e2e_gap.py 20 2>&1 | grep -v kernels)
  done
done

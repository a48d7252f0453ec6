# quick GPU loop: the posterior / forest tests, then the bench lines (args: configs)
set -x
timeout 900 python -m pytest tests/test_gpu_properties.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_quick.log 2>&1; echo tests=$?
tail -3 gpurun_out/gpu_quick.log
for c in ${@:-M200 C3}; do python bench.py --config $c --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/bench_*.json")):
    try:
        d = json.load(open(f)); r = d["roofline"]
        print(f, "%.4g" % d["value"], "e2e %.4g" % d["e2e"]["value"], {k: round(v, 3) for k, v in r["kernel_ms"].items() if k != "note"},
              "frac", r.get("datapath") and round(r["datapath"]["frac"], 3))
    except Exception as e:
        print(f, "ERR", e)
PY

#!/bin/bash
# The driver's two bench arms (N=1), as the round-end run does them.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python bench.py --gpus 1 --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --gpus 1 --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
for f in ["gpurun_out/bench.json", "gpurun_out/bench_ref.json"]:
    try:
        d = json.loads(open(f).read().splitlines()[-1])
        print(f, round(d["value"]), "e2e", round(d["e2e"]["value"]), "parity", d.get("parity_ok"),
              "roof", (d.get("roofline") or {}).get("frac"))
        print(json.dumps(d["config"].get("legs")))
    except Exception as e:
        print(f, "ERR", e)
PY
tail -n 3 gpurun_out/bench.err gpurun_out/bench_ref.err

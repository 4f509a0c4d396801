#!/bin/bash
for c in ${@:-c4 c2 c5 c1}; do timeout 300 python scripts/trace_layer.py --config $c > gpurun_out/trace_$c.json 2>&1; done
python - "$@" <<'PY'
import json, sys
for c in (sys.argv[1:] or ["c4", "c2", "c5", "c1"]):
    try:
        j = json.load(open("gpurun_out/trace_" + c + ".json"))
    except Exception:
        print(c, open("gpurun_out/trace_" + c + ".json").read()[-1500:]); continue
    print(c, "ideal", j["ideal_us_at_peak"], {k: v for k, v in j["phases_us_mean_over_ctas"].items()})
    print("   max", j["phases_us_max_over_ctas"])
    print("   issue", j["cta0_stage_issue_us"]); print("   ready", j["cta0_stage_ready_us"])
PY

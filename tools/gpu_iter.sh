#!/bin/bash
# One GPU iteration: parity tests, then the bench in both precisions.
# Usage (under gpurun): bash tools/gpu_iter.sh [pytest-args]
set -u
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -q -m gpu -x ${1:-} > gpurun_out/gputests.log 2>&1
echo "gpu tests rc=$?"; tail -5 gpurun_out/gputests.log
for prec in bf16 fp32; do
  timeout -s KILL 300 python bench.py --precision $prec --no-cpu-baseline > gpurun_out/bench_$prec.json 2> gpurun_out/bench_$prec.err
  echo "bench $prec rc=$?"
  python - "$prec" <<'EOF'
import json, sys
p = sys.argv[1]
try:
    d = json.load(open("gpurun_out/bench_%s.json" % p))
except Exception as e:
    print("no json", e); sys.exit(0)
print(p, "value %.0f e2e %.0f p50 %.3f ms" % (d["value"], d["e2e"]["value"], d["p50_frame_latency_ms"]))
print("  stages", {k: round(v, 4) for k, v in d["stage_ms"].items()})
r = d["roofline"]; print("  roofline", r["kernel"], r["bound"], "%.3g %s frac %.4f" % (r["achieved"], r["unit"], r["frac"]), "clocks", d["clocks"])
c3 = d.get("c3")
if c3: print("  c3 meshes/s %.0f full %.3f ms lbs %.3f ms %.0f GB/s frac %.3f" % (c3["meshes_per_s"], c3["ms_full"], c3["ms_lbs_fk"], c3["lbs_achieved_gbs"], c3["lbs_frac_of_hbm"]))
EOF
done

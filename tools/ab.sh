#!/bin/bash
# A/B of library variants on one box, alternating runs (experiments only).
#   tools/ab.sh OUT REPS "bench args" lib1 lib2 ...   (lib "base" = the in-tree build)
out=$1; reps=$2; args=$3; shift 3
mkdir -p gpurun_out
for rep in $(seq 1 $reps); do
  for lib in "$@"; do
    if [ "$lib" = base ]; then unset BD_LIB; else export BD_LIB=_ab/libbitdelta_$lib.so; fi
    line=$(timeout 600 python bench.py $args --no-cpu-baseline 2>gpurun_out/ab_err.log | tail -1)
    python - "$lib" "$line" >> gpurun_out/$out <<'PY'
import json, sys
lib, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
except Exception:
    print(lib, "FAILED", line[:300]); sys.exit()
dk = d.get("delta_kernel", {}).get("per_group", {})
print(lib, d["value"], d["ms_per_step"], d.get("clocks", {}).get("sm_mhz"),
      {k: v["gbs"] for k, v in dk.items()},
      {k: v for k, v in d.get("profile_ms_per_step", {}).items() if v})
PY
  done
done
cat gpurun_out/$out

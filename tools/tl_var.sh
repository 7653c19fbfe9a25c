# timeline + bench per variant (env); AB_VARS overrides
cd $GRAFT_REPO_ROOT
VARS=${TL_VARS:-"BD_LUT_STEAL=0 BD_LUT_STEAL=200"}
for v in $VARS; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout 600 python tools/timeline.py --out gpurun_out/tl_$tag.txt > /dev/null 2>&1
  echo "== $v"; grep -E "^# (lut|k2|step|time)" gpurun_out/tl_$tag.txt
done
for rep in 1 2; do for v in $VARS; do
  env $v timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/v.json')); print('$v', d['ms_per_step'])"
done; done

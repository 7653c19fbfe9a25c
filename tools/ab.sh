# A/B: alternate runs of tools/ab/lib<X>.so variants on the same box; a variant may carry env: "B:BD_KVPF=0"
cd $GRAFT_REPO_ROOT
VARS=${AB_VARS:-"A B"}
for rep in 1 2 3; do
for v in $VARS; do
lib=${v%%:*}; envs=""; [ "$v" != "$lib" ] && envs=${v#*:}
env $envs BD_LIB=$PWD/tools/ab/lib$lib.so timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
python -c "
import json;d=json.load(open('gpurun_out/v.json'));p=d.get('profile_ms_per_step',{});print('$v',d['value'],d['ms_per_step'],' '.join(f'{k}={v}' for k,v in p.items() if v))" 2>/dev/null || tail -2 gpurun_out/v.err
done; done

# L2 prefetch (glue kernels prefetch the next linear's first K2/K3 bytes): sweep
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
run() {
  timeout 300 env "$@" python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/v.json 2>gpurun_out/v.err
  python -c "
import json;d=json.load(open('gpurun_out/v.json'));p=d.get('profile_ms_per_step',{});print('$*',d['value'],d['ms_per_step'],' '.join(f'{k}={v}' for k,v in p.items() if v))" 2>/dev/null || tail -3 gpurun_out/v.err
}
run BD_PF=0
run BD_PF=1
run BD_PF_K2=2 BD_PF_K3=512
run BD_PF_K2=8 BD_PF_K3=2048
run BD_PF_K2=16 BD_PF_K3=4096
run BD_PF_K2=8 BD_PF_K3=0
run BD_PF_K2=0 BD_PF_K3=2048
run BD_PF=0

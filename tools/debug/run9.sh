run() { echo "== $*"; python bench.py --also "" --no-cpu --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print(round(d['value']), 'e2e', round(d['e2e']['value']), ' '.join(f\"{n}:{v['avg_launch_us']:.1f}us/{v['share']:.2f}\" for n,v in k.items()))"; }
run --opt stream_vcycle=0
python tools/debug/vc_classes.py 74 "" stream_vcycle=0 stream_vcycle=1,staged_legs=1 staged_legs=0
export HB_RPC_DOWN=8 HB_RPC_UP=16; run
python tools/debug/vc_classes.py 74 ""
export HB_RPC_DOWN=8 HB_RPC_UP=8; run
export HB_RPC_DOWN=4 HB_RPC_UP=16; run

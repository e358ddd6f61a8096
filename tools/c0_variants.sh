# c0 x 444 experiment sweep: one bench value per library variant (no CPU legs, no also lines)
run() { echo "== $*"; python bench.py --also "" --no-cpu --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print(round(d['value']), 'e2e', round(d['e2e']['value']), ' '.join(f\"{n}:{v['avg_launch_us']:.1f}us/{v['share']:.2f}\" for n,v in k.items()))"; }
run
run --opt coarse_reg=0
run --opt staged_legs=0
run --opt split_vcycle=0
run --groups 2
run --groups 4
HB_RPC_DOWN=8 HB_RPC_UP=16 run
HB_RPC_DOWN=16 HB_RPC_UP=32 run
HB_RPC_DOWN=2 HB_RPC_UP=4 run

run() { echo "== $*"; python bench.py --also "" --no-cpu --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print(round(d['value']), 'e2e', round(d['e2e']['value']), ' '.join(f\"{n}:{v['avg_launch_us']:.1f}us/{v['share']:.2f}\" for n,v in k.items()))"; }
for f in 8 4 2 1; do echo "fill $f"; HB_RPC_FILL=$f run; done
HB_RPC_FILL=2 run --replicas 148
HB_RPC_FILL=8 run --replicas 148

run() { python bench.py --also "" --no-cpu --no-pipeline --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print(round(d['value']), 'ms', round(d['ms_per_step'],2), ' '.join(f\"{n}:{v['avg_launch_us']:.1f}us/{v.get('hbm_frac',0):.2f}\" for n,v in k.items()))"; }
run; run
python -m pytest tests -m gpu -x -q -k "fgmres or krylov or block or c0 or converged" 2>&1 | tail -2

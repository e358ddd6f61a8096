run() { echo "== $*"; python bench.py --also "" --no-cpu --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), 'e2e', round(d['e2e']['value']))"; }
run
run --groups 2
run --groups 4
run --replicas 592 --groups 4
run --replicas 592
run --opt split_vcycle=0
run --groups 4 --opt split_vcycle=0

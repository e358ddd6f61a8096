# c0 throughput against the number of column groups and replicas per step (device / pipelined e2e / per-step-joined e2e)
run() { echo "== $*"; python bench.py --also "" --no-cpu --steps 5 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), 'e2e', round(d['e2e']['value']), 'sync', round(d['e2e'].get('per_step_sync',{}).get('value',0)), 'ms', round(d['ms_per_step'],2), d['config']['rhs_per_gpu_per_step'])"; }
run "$@" --groups 3 --replicas 1332
run "$@" --groups 3 --replicas 1776
run "$@" --groups 4 --replicas 1184
run "$@" --groups 2 --replicas 888
run "$@" --groups 3 --replicas 666
run "$@" --groups 3 --replicas 888

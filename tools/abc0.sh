#!/bin/bash
# c0 solves/s A/B: each argument is "<label>|<env and bench options>", e.g.
#   bash tools/abc0.sh "new|" "old|HB_LIB_PATH=build/ab/HEAD/libhelmgpu.so" "nofuse|--opt arnoldi=0"
for spec in "$@"; do
  lab=${spec%%|*}; rest=${spec#*|}
  envs=""; opts=""
  for w in $rest; do case $w in *=*/*|HB_*=*) envs="$envs $w";; *) opts="$opts $w";; esac; done
  env $envs python bench.py --also , --no-cpu --steps 5 $opts 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$lab', round(d['value']), round(d['e2e']['value']), d['config']['iterations'])"
done

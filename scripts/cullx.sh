for c in C2 C3; do for v in 0 1; do echo "$c CULL=$v"; APML_CULL=$v python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()}, d['gpu_launches'])"; done; done

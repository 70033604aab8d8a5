for t in 2368 1184 592 296 148; do echo "target $t"; APML_SPLIT_TARGET=$t python bench.py --no-cpu-baseline --no-e2e --steps 10 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})"; done

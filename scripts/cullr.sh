for lib in libapml_c1.so libapml.so libapml_c4.so; do for c in C4 C5; do echo "$lib $c"; APML_LIB=$PWD/paper_2512_19743_b200/$lib python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})"; done; done

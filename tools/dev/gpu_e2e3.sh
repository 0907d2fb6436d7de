for k in 1 2 3; do python bench.py --no-cpu --no-paper --steps 3 > gpurun_out/e2e3_$k.json 2>gpurun_out/e2e3_$k.err; python -c "
import json; d=json.loads(open('gpurun_out/e2e3_$k.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"; done

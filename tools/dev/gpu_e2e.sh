nvidia-smi topo -m 2>&1 | head -5
lscpu | grep -E "NUMA|^CPU\(s\)|Model name"
python tools/pcie_probe.py 2>&1 | tail -5
for k in 1 2; do python bench.py --no-cpu --no-paper > gpurun_out/e2e_$k.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/e2e_$k.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"; done

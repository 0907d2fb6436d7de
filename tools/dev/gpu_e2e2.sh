free -g | head -2
python tools/dev/e2e_probe.py 10000
python tools/dev/e2e_probe.py 10000

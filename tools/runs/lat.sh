python tools/latency_probe.py > gpurun_out/lat_after.jsonl 2>&1
python -m pytest tests/ -q -m gpu -x --timeout 900 2>&1 | tail -3

timeout 600 python -m pytest tests/test_gpu_discrete.py -m gpu -x -q --timeout 300 -k "HostStreaming" 2>&1 | tail -2
python bench.py --no-soft --no-ns --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"

timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -1
for i in 1 2; do timeout 100 python tools/quick_bench.py 2>&1 | grep hist; done
echo done

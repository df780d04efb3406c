timeout 600 python -m pytest tests/test_gpu_discrete.py -m gpu -x -q --timeout 300 2>&1 | tail -1
for M in default cta; do echo "== $M"; ECC_B200_F3=$M timeout 100 python tools/quick_bench.py 2>&1 | grep hist; done
echo done

timeout 900 python -m pytest tests/test_gpu_discrete.py tests/test_cli.py tests/test_io.py -m gpu -x -q --timeout 600 2>&1 | tail -2
for M in default rank2; do echo "== $M"; ECC_B200_F3=$M timeout 100 python tools/quick_bench.py 2>&1 | grep hist; done
echo done

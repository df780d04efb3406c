timeout 600 python -m pytest tests/test_gpu_discrete.py tests/test_cli.py tests/test_io.py -m gpu -x -q --timeout 300 2>&1 | tail -1
for i in 1 2; do timeout 100 python tools/quick_bench.py 2>&1 | grep hist; done
python tools/prof_discrete.py 512 2 >/dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fast3d -s 1 -c 1 -o gpurun_out/prof_rank python tools/prof_discrete.py 512 2 > /dev/null 2>&1
echo done

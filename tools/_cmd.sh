timeout 600 python -m pytest tests/test_gpu_soft.py -m gpu -x -q --timeout 300 2>&1 | tail -1
timeout 100 python tools/quick_bench.py 2>&1 | grep soft
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_soft16d.csv python tools/prof_soft.py 16 3 > /dev/null 2>&1
echo done

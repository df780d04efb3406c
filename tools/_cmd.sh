timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_soft3d_b.csv python tools/prof_soft3d.py 512 1 > /dev/null 2>&1
ECC_B200_GENERIC=1 timeout 100 python tools/quick_bench.py 2>&1 | grep hist
echo done

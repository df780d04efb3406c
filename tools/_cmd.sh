timeout 600 python -m pytest tests/test_gpu_soft.py tests/test_gpu_discrete.py -m gpu -x -q --timeout 300 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_soft16d.csv python tools/prof_soft.py 16 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:soft_prep2d -s 1 -c 1 -o gpurun_out/prof_prep python tools/prof_soft.py 16 2 > /dev/null 2>&1
echo done

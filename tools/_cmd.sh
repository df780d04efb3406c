timeout 600 python -m pytest tests/test_gpu_soft.py -m gpu -x -q --timeout 300 2>&1 | tail -1
ECC_SOFT_FWD_T=8 ECC_SOFT_BWD_T=8 timeout 600 python -m pytest tests/test_gpu_soft.py -m gpu -x -q --timeout 300 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t16.csv python tools/prof_soft.py 16 3 > /dev/null 2>&1
ECC_SOFT_FWD_T=8 ECC_SOFT_BWD_T=8 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t8.csv python tools/prof_soft.py 16 3 > /dev/null 2>&1
echo done

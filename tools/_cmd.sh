timeout 600 python -m pytest tests/test_gpu_soft.py -m gpu -x -q --timeout 300 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none -k regex:ecc_soft_kernel -c 2 python tools/prof_soft.py 16 2 2>&1 | grep -E "duration|pipe"

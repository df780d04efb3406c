python bench.py > gpurun_out/bench_r01h.json 2> gpurun_out/bench_r01h.err; tail -1 gpurun_out/bench_r01h.json | cut -c1-300
python tools/prof_discrete.py 512 2 >/dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fast3d -s 1 -c 1 -o gpurun_out/prof_rank_ws python tools/prof_discrete.py 512 2 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
python tools/prof_discrete.py 1024 2 >/dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --clock-control none -k regex:fast3d -s 1 -c 1 python tools/prof_discrete.py 1024 2 2>&1 | grep -E "duration|dram|wavefronts"
echo done

python bench.py > gpurun_out/bench_r01d.json 2> gpurun_out/bench_r01d.err; tail -1 gpurun_out/bench_r01d.json
python tools/prof_discrete.py 512 2 >/dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fast3d -s 1 -c 1 -o gpurun_out/prof_bin_v1 python tools/prof_discrete.py 512 2 > gpurun_out/ncu9.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json
echo done

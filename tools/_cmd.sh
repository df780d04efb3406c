python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -1
python bench.py > gpurun_out/bench_r01k.json 2> gpurun_out/bench_r01k.err; tail -1 gpurun_out/bench_r01k.json | cut -c1-150
python bench.py --impl reference > gpurun_out/bench_ref_k.json 2>/dev/null; tail -1 gpurun_out/bench_ref_k.json | cut -c1-150
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-ns > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_soft16f.csv python tools/prof_soft.py 16 3 > /dev/null 2>&1
echo done

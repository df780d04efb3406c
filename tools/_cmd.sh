timeout 300 python tools/prof_soft3d.py 1024 1 2>&1 | tail -1
timeout 300 python tools/prof_soft3d.py 512 2 2>&1 | tail -1
python bench.py > gpurun_out/bench_r01e.json 2> gpurun_out/bench_r01e.err; tail -1 gpurun_out/bench_r01e.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['soft']['value'], d['soft']['ms_per_step'], d['e2e']['value'])"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_soft3d.csv python tools/prof_soft3d.py 512 1 > /dev/null 2>&1
echo done

python tools/prof_discrete.py 512 2 >/dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:fast3d -s 1 -c 1 -o gpurun_out/prof_edge python tools/prof_discrete.py 512 2 > /dev/null 2>&1
echo done

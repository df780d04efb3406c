for V in "-DECC_BWD_PACKED=1 -DECC_EMU_BWD=0" "-DECC_BWD_PACKED=1 -DECC_EMU_BWD=1" "-DECC_BWD_PACKED=1 -DECC_EMU_BWD=2"; do
  ECC_B200_NVCC_EXTRA="$V" python -c "from paper_2510_20271_b200.build import build; build(force=True)" > /dev/null 2>&1
  N=$(echo $V | tr -dc '0-9')
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/emub_$N.csv python tools/prof_soft.py 16 3 > /dev/null 2>&1
done
python -c "from paper_2510_20271_b200.build import build; build(force=True)" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ecc_soft_kernel<1" -s 1 -c 1 -o gpurun_out/prof_bwd16 python tools/prof_soft.py 16 2 > /dev/null 2>&1
echo done

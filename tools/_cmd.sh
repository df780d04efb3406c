for F in 2 3 4; do
  ECC_B200_NVCC_EXTRA="-DECC_EMU_FWD=$F" python -c "from paper_2510_20271_b200.build import build; build(force=True)" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/emuf_$F.csv python tools/prof_soft.py 16 3 > /dev/null 2>&1
done
echo done

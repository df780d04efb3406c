for V in 16 32 64; do
  ECC_B200_NVCC_EXTRA="-DPREP_TH=$V" python -c "from paper_2510_20271_b200.build import build; build(force=True)" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:soft_prep2d -c 3 python tools/prof_soft.py 16 2 2>&1 | grep duration | head -3 | sed "s/^/TH=$V /"
done

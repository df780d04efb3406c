for V in 0 1 2; do
  ECC_B200_NVCC_EXTRA="-DECC_SOFT_EX2_FMA=$V" python -c "from paper_2510_20271_b200.build import build; build(force=True)" > /dev/null 2>&1
  echo "== $V"; timeout 600 python -m pytest tests/test_gpu_soft.py -m gpu -x -q --timeout 300 2>&1 | tail -1
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:ecc_soft_kernel -c 2 python tools/prof_soft.py 16 2 2>&1 | grep -E "duration"
done

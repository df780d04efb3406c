for V in 3 4; do
  ECC_B200_NVCC_EXTRA="-DECC_F3_MINB=$V" python -c "from paper_2510_20271_b200.build import build; build(force=True)" > /dev/null 2>&1
  echo "== minb $V"; timeout 100 python tools/quick_bench.py 2>&1 | grep hist
done

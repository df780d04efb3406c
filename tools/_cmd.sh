for V in "-DECC_F3_FMA_PP=0" "-DECC_F3_FMA_PP=1" "-DECC_F3_FMA_TR=1" "-DECC_F3_FMA_DEP=1"; do
  ECC_B200_NVCC_EXTRA="$V" python -c "from paper_2510_20271_b200.build import build; build(force=True)" > /dev/null 2>&1
  echo "== $V"; timeout 100 python tools/quick_bench.py 2>&1 | grep hist
done

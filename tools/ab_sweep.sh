for v in 600 2400; do
  python tools/ab_env.py 4 4096 32 DTN_GEMM_BIG_TILES=$v
  python tools/ab_env.py 2 512 16 DTN_GEMM_BIG_TILES=$v
done

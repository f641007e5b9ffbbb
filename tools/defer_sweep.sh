for t in 1e7 3.2e7 1e8; do
  DTN_DEFER_MIN_WORK=$t python tools/defer_check.py 4 4096 32 | sed "s/^/thr $t: /"
done
for c in "2 512 16" "3 1024 32" "5 2048 32"; do
  python tools/defer_check.py $c | sed "s/^/default: /"
done

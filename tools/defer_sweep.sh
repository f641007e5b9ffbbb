for c in "4 4096 32" "5 2048 32"; do
  DTN_DEFER_MIN_WORK=1 python tools/defer_check.py $c | sed "s/^/forced: /"
  python tools/defer_check.py $c | sed "s/^/default: /"
done
DTN_DEFER_MIN_WORK=1 python tools/defer_check.py 2 512 16 | sed "s/^/forced: /"

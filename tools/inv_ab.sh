python tools/build_overhead.py 2>&1 | grep "^2 host" | tail -2
DTN_INV_SWEEP=1 python tools/build_overhead.py 2>&1 | grep "^2 host" | tail -2

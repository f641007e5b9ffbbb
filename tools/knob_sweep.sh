# cfg2 build time (graph, with G) under the engine's schedule knobs
for env in "" "DTN_FAST_THRESHOLD=1" "DTN_FAST_THRESHOLD=2" "DTN_FAST_THRESHOLD=4"; do
  echo "== $env"; env $env python tools/build_overhead.py 2>&1 | grep "^2 host" | tail -2
done

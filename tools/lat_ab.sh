# same-box A/B of the latency regime: bash tools/lat_ab.sh CONFIG LIB...  (TOOL)
CFG=$1; shift
for L in "$@"; do QVG_LIB=$L python bench.py --config $CFG --steps 5 --sweep none --relaxed none --batch-sizes 1,128,1024 --rerank-depths none --no-cpu-baseline --recall-queries 0 --variant-rows none > /tmp/lat.json 2>/tmp/lat.err || tail -3 /tmp/lat.err; python -c "
import json,sys; d=json.loads(open('/tmp/lat.json').read()); print('$L', [(r['batch'], round(r['p50_ms'],4), r['parity']['ids_identical']) for r in d['batch_latency']])"; done

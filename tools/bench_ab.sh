# same-box A/B of bench.py lines: bash tools/bench_ab.sh "ARGS" LIB1 LIB2 ...  (TOOL)
ARGS=$1; shift
for L in "$@"; do
  QVG_LIB=$L python bench.py $ARGS --no-cpu-baseline --recall-queries 0 --sweep none --relaxed none > /tmp/ab.json 2>/tmp/ab.err || tail -3 /tmp/ab.err
  python -c "
import json; d=json.load(open('/tmp/ab.json'))
print('$L', 'value %.4fM e2e %.4fM kernel %.4f ms frac %.3f evals exact %.1f lossy %.1f' % (d['value']/1e6, d['e2e']['value']/1e6, d['roofline']['kernel_ms'], d['roofline']['frac'], d['counters']['evals_per_query_exact'], d['counters']['evals_per_query_lossy']))"
done

# same-box A/B of bench.py lines with parity: bash tools/ab.sh "ARGS" LIB1 LIB2 ...  (TOOL)
ARGS=$1; shift
for L in "$@"; do
  QVG_LIB=$L timeout 600 python bench.py $ARGS --no-cpu-baseline --recall-queries 0 --relaxed none --variant-rows none > /tmp/ab.json 2>/tmp/ab.err || tail -3 /tmp/ab.err
  python - "$L" <<'P'
import json, sys
d = json.load(open('/tmp/ab.json'))
p = d.get('parity', {})
pd = p.get('timed_device', {})
pe = p.get('timed_e2e', {})
print(sys.argv[1], 'value %.4fM e2e %.4fM kernel %.4f ms frac %.3f | parity dev %s/%s e2e %s/%s' % (
    d['value'] / 1e6, d['e2e']['value'] / 1e6, d['roofline']['kernel_ms'], d['roofline']['frac'],
    pd.get('ids_identical'), pd.get('scores_bit_identical'), pe.get('ids_identical'),
    pe.get('scores_bit_identical')))
for r in d.get('ef_sweep', []):
    print('   ef %d: %.4fM qps kernel %.4f ms frac %.3f parity %s' % (
        r['ef'], r['qps'] / 1e6, r['kernel_ms'], r['frac'], r.get('parity', {}).get('ids_identical')))
for r in d.get('batch_latency', []):
    print('   batch %d: p50 %.4f ms p99 %.4f ms parity %s' % (
        r['batch'], r['p50_ms'], r['p99_ms'], r.get('parity', {}).get('ids_identical')))
P
done

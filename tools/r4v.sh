# final-tree measurement (with tail balancing): GPU tests, cfg1 / cfg1-norm bench lines, launch list and
# full ncu captures (headline kernel ef 64 / 256, cfg1-norm, latency kernel batch 1), each
# capture only after its plain run exited 0
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r4v_gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r4v_gputests.log
timeout 600 python bench.py --config 1 --out gpurun_out/r4v_bench_cfg1.json > gpurun_out/r4v_bench_cfg1.log 2>&1; echo "cfg1 rc=$?"
timeout 600 python bench.py --config 1 --sigma-mode norm --relaxed 2,4 --out gpurun_out/r4v_bench_cfg1n.json > gpurun_out/r4v_bench_cfg1n.log 2>&1; echo "cfg1n rc=$?"
P="python tools/one_launch.py"
cap() { # name kernel-regex args...
  local name=$1 rx=$2; shift 2
  $P "$@" > gpurun_out/p_$name.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 1 -c 1 -o gpurun_out/r4v_$name $P "$@" > gpurun_out/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
}
cap cfg2 search_kernel 2 10000 64 dev
cap cfg2_ef256 search_kernel 2 10000 256 dev
cap cfg1n search_kernel 1 10000 64 dev norm
cap coop_b1 coop_kernel 2 1 64 dev
timeout 600 python bench.py --steps 2 --warmup 3 --sweep none --relaxed none --no-cpu-baseline --recall-queries 0 > gpurun_out/b2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r4v_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --sweep none --relaxed none --no-cpu-baseline --recall-queries 0 > gpurun_out/ncu_l.log 2>&1; echo "launch list rc=$?"
for f in cfg1 cfg1n; do python - $f <<'PY'
import json, sys
d = json.load(open(f'gpurun_out/r4v_bench_{sys.argv[1]}.json'))
print(sys.argv[1], 'value %.3fM e2e %.3fM kernel %.4f frac %.3f' % (d['value']/1e6, d['e2e']['value']/1e6, d['roofline']['kernel_ms'], d['roofline']['frac']), d['counters'], d['parity']['timed_device'], d.get('recall_at_10'), d['cpu_baseline'].get('value'))
for r in d.get('relaxed', []): print('  relaxed', r['expansions_per_step'], round(r['qps']), r['recall_at_10'], r['exact_recall_at_10'])
PY
done

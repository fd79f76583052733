# round-2 measurement of the r2h kernels: cfg1 / cfg1-norm / cfg2 bench lines, launch list
# and one full ncu capture of the headline kernel (each only after its plain run exited 0)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py --out gpurun_out/r2h_bench_cfg2.json > gpurun_out/r2h_bench_cfg2.log 2>&1; echo "cfg2 rc=$?"
timeout 600 python bench.py --config 1 --out gpurun_out/r2h_bench_cfg1.json > gpurun_out/r2h_bench_cfg1.log 2>&1; echo "cfg1 rc=$?"
timeout 600 python bench.py --config 1 --sigma-mode norm --relaxed 2,4 --out gpurun_out/r2h_bench_cfg1n.json > gpurun_out/r2h_bench_cfg1n.log 2>&1; echo "cfg1n rc=$?"
P="python tools/one_launch.py"
$P 2 10000 64 dev > gpurun_out/p_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 -o gpurun_out/r2h_cfg2 $P 2 10000 64 dev > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --sweep none --relaxed none --no-cpu-baseline --recall-queries 0 > gpurun_out/b2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2h_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --sweep none --relaxed none --no-cpu-baseline --recall-queries 0 > gpurun_out/ncu_l.log 2>&1; echo "launch list rc=$?"
for f in cfg2 cfg1 cfg1n; do python - $f <<'P'
import json, sys
d = json.load(open(f'gpurun_out/r2h_bench_{sys.argv[1]}.json'))
print(sys.argv[1], 'value %.3fM e2e %.3fM kernel %.4f frac %.3f' % (d['value']/1e6, d['e2e']['value']/1e6, d['roofline']['kernel_ms'], d['roofline']['frac']), d['counters'], d['parity']['timed_device'], d.get('recall_at_10'))
P
done

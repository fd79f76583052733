# round-2 re-entry measurement on HEAD: GPU tests, headline bench, contender
# counts (tail build) and per-phase cycles (phases build)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2d_gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r2d_gputests.log
timeout 900 python bench.py --out gpurun_out/r2d_bench_cfg2.json > gpurun_out/r2d_bench.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/r2d_bench_cfg2.json
for ef in 64 256; do
  QVG_LIB=build/tail/libqvg.so timeout 300 python tools/tail_profile.py 2 $ef > gpurun_out/r2d_tail_ef$ef.log 2>&1
  cat gpurun_out/r2d_tail_ef$ef.log | tail -8
done
QVG_LIB=build/phases/libqvg.so timeout 300 python tools/phase_times.py 2 > gpurun_out/r2d_phases.log 2>&1
cat gpurun_out/r2d_phases.log | tail -12

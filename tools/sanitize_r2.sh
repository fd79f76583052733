# usage: bash tools/sanitize_r2.sh TOOL   (one compute-sanitizer tool per gpurun call)
T=$1
S="/usr/local/cuda/bin/compute-sanitizer --tool $T --error-exitcode 9"
[ "$T" = racecheck ] && S="$S --racecheck-report all"
python tools/sanitize_run.py geo > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
for w in geo coop relp pipe one build; do
  if [ $w = geo ]; then E="QVG_COOP_MAX_NQ=0"; else E=""; fi
  env $E timeout 900 $S python tools/sanitize_run.py $w > gpurun_out/san_${T}_$w.log 2>&1
  echo "$T $w rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|identical|MISMATCH|ran|ok' gpurun_out/san_${T}_$w.log | tr '\n' ' ')"
done

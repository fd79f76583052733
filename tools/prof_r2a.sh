set -e
P="python tools/one_launch.py"
$P 1 10000 64 dev norm > gpurun_out/p_c1n.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 -o gpurun_out/r2_cfg1n $P 1 10000 64 dev norm > gpurun_out/ncu_c1n.log 2>&1
$P 1 10000 64 dev literal > gpurun_out/p_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 -o gpurun_out/r2_cfg1 $P 1 10000 64 dev literal > gpurun_out/ncu_c1.log 2>&1
$P 2 10000 256 dev > gpurun_out/p_c2e256.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 1 -c 1 -o gpurun_out/r2_cfg2_ef256 $P 2 10000 256 dev > gpurun_out/ncu_c2e256.log 2>&1
$P 2 1 64 dev > gpurun_out/p_coop.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:coop_kernel -s 1 -c 1 -o gpurun_out/r2_coop_b1 $P 2 1 64 dev > gpurun_out/ncu_coop.log 2>&1
$P 2 128 64 dev > gpurun_out/p_coop128.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:coop_kernel -s 1 -c 1 -o gpurun_out/r2_coop_b128 $P 2 128 64 dev > gpurun_out/ncu_coop128.log 2>&1
ls -la gpurun_out/*.ncu-rep

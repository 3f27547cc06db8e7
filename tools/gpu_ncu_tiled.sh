CMD="python tools/perm_bench.py 192"
$CMD > gpurun_out/plain_pb.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:permute_tiled -s 3 -c 1 -o gpurun_out/prof_tiled_$1 $CMD > gpurun_out/ncu_tiled.log 2>&1; echo "ncu rc=$?"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:permute_rows -s 16 -c 1 -o gpurun_out/prof_rows_$1 $CMD > gpurun_out/ncu_rows.log 2>&1; echo "ncu rc=$?"

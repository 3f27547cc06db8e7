TK_SVD_DEBUG=1 timeout 300 python tools/bench_svd.py --reps 1 > gpurun_out/r2f_svd_dbg.txt 2>&1; echo "svd dbg rc=$?"
grep "tk svd" gpurun_out/r2f_svd_dbg.txt | sed 's/.*block [0-9]*: //' | sort -u | sort -n | awk '!seen[$1" "$3" "$5]++' | awk 'NR%5==0'

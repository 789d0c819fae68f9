mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_read_lookup_miss.sum
for v in q64 t64; do for f in 2 8 130; do
LRB_DEBUG_FLAGS=$f timeout 300 ncu --metrics $M --clock-control none -k regex:lrb_gemm_kernel -c 1 --csv python tools/profile_one.py --config cfg2 --variant $v --launches 1 > gpurun_out/ncu_l2b_${v}_$f.csv 2>&1
done; done
for f in gpurun_out/ncu_l2b_*.csv; do echo $f; grep -E "dram__|lts__|gpu__time" $f | awk -F, '{print $(NF-2), $NF}'; done

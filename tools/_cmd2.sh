mkdir -p gpurun_out
python tools/probe_policy.py cfg2 q64,t64,sq,n64 0,32,128,4 > gpurun_out/policy_cfg2.jsonl 2>&1
python tools/probe_policy.py cfg3_b1024_r32 n32,t64 0,32,128 >> gpurun_out/policy_cfg2.jsonl 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_read_lookup_miss.sum,lts__t_sectors_op_write.sum
for v in q64 t64 sq; do for f in 0 32; do
LRB_DEBUG_FLAGS=$f timeout 300 ncu --metrics $M --clock-control none -k regex:lrb_gemm_kernel -c 1 --csv python tools/profile_one.py --config cfg2 --variant $v --launches 1 > gpurun_out/ncu_l2_${v}_$f.csv 2>&1
done; done

set -x
mkdir -p gpurun_out/prof2 data_cfg2
oracle/_ref/fsi_ref_harness export cfg2 data_cfg2/cfg2.fsix --no-mult --no-gmres > gpurun_out/prof2/export.log 2>&1
export FSI_DATA=data_cfg2/cfg2.fsix FSI_MAXIT=30
for k in k_update_dots_norm k_update_normalize k_spmv_dots_s prolong_resid_pair_kernel; do
  timeout 400 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:$k --launch-skip 12 -c 1 -o /tmp/p_$k python tools/profile_solve.py solve > gpurun_out/prof2/ncu_$k.log 2>&1
  ncu -i /tmp/p_$k.ncu-rep --page details --csv > /tmp/d.csv 2>&1
  grep -E '"(Duration|DRAM Throughput|Memory Throughput|L1/TEX Cache Throughput|L2 Cache Throughput|Achieved Occupancy|Theoretical Occupancy|Registers Per Thread|L1/TEX Hit Rate|L2 Hit Rate|Executed Ipc Active|Eligible Warps Per Scheduler|Waves Per SM|Block Limit Registers|Block Limit Shared Mem)' /tmp/d.csv | awk -F'","' '{print $(NF-3)" | "$(NF-2)" | "$(NF-1)" | "$NF}' | sort -u > gpurun_out/prof2/${k}_summary.txt
  python tools/ncu_lines.py /tmp/p_$k.ncu-rep 25 > gpurun_out/prof2/${k}_lines.txt 2>&1
done
du -sh gpurun_out

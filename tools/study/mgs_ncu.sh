cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cc in all none; do
ncu --cache-control $cc --clock-control none -k regex:mgs_bulk -s 89 -c 1 --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read.sum tools/mgs_bench_bin 5451776 30 2>&1 | grep -E "gpu__|dram__|lts__" | sed "s/^/$cc /"
done | tee gpurun_out/mgs_ncu.txt
L2P=1.0 tools/mgs_bench_bin 5451776 30 | tee -a gpurun_out/mgs_ncu.txt

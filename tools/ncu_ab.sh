mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in base FUSED0 RG64; do
  case $v in base) E="";; RG64) E="STARSD_RGROUP=64";; esac
  env $E timeout 900 ncu --set full --clock-control none -k regex:"k_row_stats|k_sample" -s 10 -c 2 -f -o gpurun_out/ab_full_c3_$v python tools/profile_run.py --config c3 --calls 16 > gpurun_out/ab_ncu_$v.log 2>&1
  ncu -i gpurun_out/ab_full_c3_$v.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size > gpurun_out/ab_raw_$v.csv 2>&1
done

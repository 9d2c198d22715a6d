# Lanczos vs bare product on C3: DRAM bytes per pJDS launch with warm caches (ncu --cache-control none)
mkdir -p gpurun_out
ncu --cache-control none --clock-control none -k regex:pjds_spmv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --csv python tools/lanczos_bench.py C3 6 > gpurun_out/ncu62_lz_c3.csv 2> gpurun_out/ncu62.err
tail -n 3 gpurun_out/ncu62.err

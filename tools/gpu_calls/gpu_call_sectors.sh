M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum
python bench.py --config C3 --steps 50 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
ncu --metrics $M --clock-control none -k regex:spmv_kernel --csv --log-file gpurun_out/sect_c3.csv python tools/kbench.py --configs C3 --dtypes f64,f32 --fmts pjds32s,pjds64s,pjds128s,pjds32,ellr --sigmas 0,16384,262144,4194304 --once > gpurun_out/sect_c3.log 2>&1
ncu --metrics $M --clock-control none -k regex:spmv_kernel --csv --log-file gpurun_out/sect_c5.csv python tools/kbench.py --configs C5 --dtypes f64 --fmts pjds32s,pjds128s --sigmas 0,262144,4194304 --once > gpurun_out/sect_c5.log 2>&1

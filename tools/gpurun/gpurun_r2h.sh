cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_atom.sum,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:"^k_commit$" -c 40 --csv --log-file gpurun_out/h_commit_steps.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/h_ncu_commit.log 2>&1; echo "ncu commit rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"^k_chain_probe$" -c 40 --csv --log-file gpurun_out/h_probe_steps.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/h_ncu_probe.log 2>&1; echo "ncu probe rc=$?"

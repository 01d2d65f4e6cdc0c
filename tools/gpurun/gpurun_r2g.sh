cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_hash_scan16|k_chain_probe|k_commit|k_epoch_fused|k_record_finish" -s 10 -c 5 -o gpurun_out/g_cfg1 python tools/config1_latency.py --reps 2 > gpurun_out/g_ncu_cfg1.log 2>&1; echo "ncu cfg1 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_atom.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_commit<" --csv --log-file gpurun_out/g_commit_steps.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/g_ncu_commit.log 2>&1; echo "ncu commit rc=$?"

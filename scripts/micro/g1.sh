mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv,noheader > gpurun_out/g1.log
timeout 300 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum,gpu__time_duration.sum --csv scripts/micro/lds_conflicts > gpurun_out/g1_micro.csv 2>&1
timeout 600 python bench.py --steps 200 --warmup 10 --no-cpu-baseline >> gpurun_out/g1.log 2>&1

#!/bin/bash
# Per-M pipe / occupancy / spill / HBM counters of the demod kernel on one C4 2048² frame
# (second launch of tools/one_launch.py, 2 frames).  Writes gpurun_out/c4_ncu_M<M>.csv.
MET=gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum,sass__inst_executed_local_loads,sass__inst_executed_local_stores,smsp__inst_executed.sum
for M in ${SIZES:-8 9 11 12 15 16 17 20 24 28 32}; do
  ncu --metrics $MET --clock-control none -k regex:demod -s 1 -c 1 --csv --log-file gpurun_out/c4_ncu_M$M.csv \
      python tools/one_launch.py --M $M --frames 2 > /dev/null 2>&1
done

# GPU-box helper: SURVEY §8(d) per-config measurements (tools/bench_configs.py) and the cfg5 ncu sweep.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python tools/bench_configs.py ${ONLY:+--only $ONLY} > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?" >> gpurun_out/configs.err
if [ -z "$NO_NCU" ]; then
timeout 600 python tools/bench_configs.py --ncu-sweep > gpurun_out/cfg5_sizes.jsonl 2> gpurun_out/cfg5_plain.err || { echo "plain sweep failed"; exit 1; }
timeout 1500 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/cfg5_ncu.csv python tools/bench_configs.py --ncu-sweep > gpurun_out/cfg5_ncu_sizes.jsonl 2> gpurun_out/cfg5_ncu.err
python tools/ncu_sweep_parse.py gpurun_out/cfg5_ncu.csv gpurun_out/cfg5_ncu_sizes.jsonl > gpurun_out/cfg5_ncu.json 2>> gpurun_out/cfg5_ncu.err
fi
echo done

# GPU-box helper: ncu --set full of one launch of each named kernel in the tracking loop
# (after the same command exited 0 without ncu), plus the launch list of 2 graph-replayed frames.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-p}
KREGEX=${2:-"k_blend_track|k_backward_track_w"}
NCAP=${3:-2}
NSKIP=${4:-20}
CMD="python bench.py --steps 2 --warmup 1 --no-mapping --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$KREGEX" -s $NSKIP -c $NCAP \
  -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
  --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo done

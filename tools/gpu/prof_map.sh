# GPU-box helper: ncu --set full of the mapping kernels of one sliding_ba view (16-keyframe window,
# ~1M Gaussians, tools/profile_map.py): after the 16 keyframe renders (32 matching launches), view 0's
# k_preprocess<1>, k_blend<2>, k_backward<2,10>, k_chain<10,1> -> gpurun_out/${TAG}_map.ncu-rep
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-pm}
timeout 900 ncu --set full --clock-control none --import-source on \
  -k "regex:^(k_chain|k_backward_q|k_pair_combine|k_blend_mq|k_preprocess)$" --launch-skip 16 -c 5 \
  -o gpurun_out/${TAG}_map python tools/profile_map.py 1 > gpurun_out/${TAG}_map.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_map.log

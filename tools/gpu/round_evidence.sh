# GPU-box helper: the round's evidence in one call — full GPU test suite, the default bench line,
# the tracking launch list + ncu --set full of the two tile kernels, and the mapping kernels' ncu.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-ev}
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
bash tools/gpu/prof.sh ${TAG}t "k_blend_track|k_backward_track_w|k_preprocess|k_tile_sort" 4 400
TAG=${TAG} bash tools/gpu/prof_map.sh
echo done

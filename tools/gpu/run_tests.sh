# GPU-box helper: the -m gpu suite (verbose, with the scale tests' printed errors) + one bench line.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-t}
nproc > gpurun_out/${TAG}_nproc.txt; lscpu | grep "Model name" >> gpurun_out/${TAG}_nproc.txt
timeout 2400 python -m pytest tests -m gpu -q -s -rA -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
fi

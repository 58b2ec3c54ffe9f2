# GPU-box helper: a pytest subset (PYTEST_K) against the in-tree library, then alternating mapping A/B
# bench runs of the variant libraries in VARIANTS, REPS times -> gpurun_out/${TAG}_abm.txt
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${TAG:-abm}
if [ -n "$PYTEST_K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$PYTEST_K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
fi
for r in $(seq 1 ${REPS:-2}); do
  bash tools/abmap.sh $VARIANTS >> gpurun_out/${TAG}_abm.txt 2>&1
done

# compute-sanitizer on the exact F345 plane-loader pipeline (and the rest of
# sanitize_small.py's runs)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export FUSEPLAN_PIPE_SEGS=3
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1200 compute-sanitizer --tool $tool --kernel-name kns=k_chain_pair python scripts/sanitize_small.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Invalid|^[0-9]" | sort | uniq -c | head -20
done

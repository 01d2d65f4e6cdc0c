cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/config1_latency.py > gpurun_out/b_cfg1_latency.json 2> gpurun_out/b_cfg1_latency.err
echo "cfg1 rc=$?"
timeout 300 python tools/step_timeline.py > gpurun_out/b_step_timeline.txt 2>&1
echo "timeline rc=$?"
WORKLOADS="1 3 4 5 6" bash tools/run_workloads.sh
for f in gpurun_out/wl*.json; do mv $f gpurun_out/b_$(basename $f); done
bash tools/sanitize.sh > gpurun_out/b_sanitize_summary.txt 2>&1
for t in memcheck racecheck synccheck initcheck; do mv gpurun_out/sanitize_$t.log gpurun_out/b_sanitize_$t.log; done
cat gpurun_out/b_sanitize_summary.txt

cd $GRAFT_REPO_ROOT
for m in 0 1 2; do
  ./tools/probe/ringrace $m 4096 > gpurun_out/ringrace_plain_$m.txt 2>&1
  timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard ./tools/probe/ringrace $m 64 > gpurun_out/racecheck_ring_mode$m.log 2>&1
  echo "mode $m rc=$?"; tail -3 gpurun_out/racecheck_ring_mode$m.log; cat gpurun_out/ringrace_plain_$m.txt
done

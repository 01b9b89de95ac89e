#!/bin/bash
# compute-sanitizer over the path's kernels on TOY shapes:
# racecheck (shared-memory hazards), synccheck (barrier misuse), memcheck
# (out-of-bounds / misaligned accesses) on K1 (exact mode and plain), its
# fix-ups, K2-K4, the K5 PDL chain (graph off and on), the prefill and the
# float32 seam.  Summaries -> gpurun_out/sanitize_<tool>.txt
O=${O:-gpurun_out}
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_run.py > $O/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> $O/sanitize_summary.txt
  tail -3 $O/sanitize_$tool.txt >> $O/sanitize_summary.txt
done

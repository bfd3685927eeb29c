cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-san}; mkdir -p $O
timeout 300 python tools/sanitize_case.py > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > $O/$tool.log 2>&1
  echo "$tool rc=$?" >> $O/$tool.log
done
grep -H "ERROR SUMMARY\|rc=\|sanitize case" $O/*.log

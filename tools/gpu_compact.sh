# compaction at 2^30: phase split (0 % fired ~ phase 1 + barrier) and a source-level ncu capture
python __graft_entry__.py > /dev/null
timeout 300 python tools/prof_scan.py 0.0 0.15 0.5 2>&1 | grep compaction
timeout 600 ncu --set full --clock-control none --import-source on -k regex:compact_fired -s 1 -c 1 -o gpurun_out/prof_compact python tools/prof_scan.py 0.15 > gpurun_out/ncu_compact.log 2>&1
echo "ncu rc=$?"

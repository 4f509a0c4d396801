python paper_2312_12456_b200/build.py > /dev/null
for a in "layer 0 1 256 1000 64" "group 148 1 256 1000 64" "group 74 2 256 1000 64" "group 8 2 256 1000 64" "group 2 1 256 1000 64" "group 2 5 256 1000 64" "group 1 1 256 1000 64" "group 1 5 256 1000 64" "group 5 1 256 1000 64"; do
  CUDA_LAUNCH_BLOCKING=1 timeout 120 python scripts/dbg/group_dbg.py $a 2>&1 | grep -E "OK|MISMATCH|Error|error" | tail -2
done

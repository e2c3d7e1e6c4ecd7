mkdir -p gpurun_out
for cfg in 0 1 2 3; do
 for split in 1 2; do
  echo "cfg=$cfg split=$split $(CRYS_SCAN_CFG=$cfg CRYS_SPLIT=$split timeout 300 python tools/split_probe.py --child --sf 20 --reps 5 2>&1 | tail -1)"
 done
done > gpurun_out/scan_sweep.txt 2>&1
cat gpurun_out/scan_sweep.txt

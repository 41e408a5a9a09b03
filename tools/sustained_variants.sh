O=gpurun_out/sus1; mkdir -p $O
for t in 4,2,4,4,1 4,2,4,1,1 4,2,3,1,1 4,2,4,0,1 4,2,5,5,1 4,2,4,2,1 4,2,4,3,1 4,2,3,3,1 4,2,3,4,1 8,2,3,1,1 4,2,3,0,1 4,2,5,0,1 4,2,4,4,1; do
  SFDB200_TILE=$t SFDB200_ZCHUNKS=5 timeout 300 python tools/step_time.py --workload cfg2 --time-steps 1000 --reps 6 >> $O/sustained_cfg2.jsonl 2>> $O/err.txt
done

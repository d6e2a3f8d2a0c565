for s in "1 4096 4096" "32 4096 4096" "128 1024 1024" "128 2048 8192" "128 16384 4096" "128 4096 16384" "64 800 320" "128 512 512" "512 1024 1024" "2048 1024 4096" "4096 11008 4096"; do
  set -- $s
  for c in auto sk 32x1 64x4 128x2; do
    if [ $c = auto ]; then unset Q8G_TC_CFG; else export Q8G_TC_CFG=$c; fi
    python tools/tc_sweep.py --m $1 --n $2 --k $3 --only "requant+rowsum" --reps 3 2>&1 | tail -1 | cut -c1-95
  done
done

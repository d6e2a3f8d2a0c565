for m in 192 256 384 512 768 1024 1536; do
  for c in auto sk 128x2 64x4; do
    if [ $c = auto ]; then unset Q8G_TC_CFG; else export Q8G_TC_CFG=$c; fi
    python tools/tc_sweep.py --m $m --only "requant+rowsum" --reps 3 2>&1 | tail -1 | cut -c1-90
  done
done

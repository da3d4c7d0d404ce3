# Synchronous pageable staging: per view (mode 0), one batch (1), chunk-pipelined (2)
set -u
for t in 14 6; do
  for m in 0 1 2; do
    for c in 1 4; do
      [ $m != 2 ] && [ $c = 1 ] && continue
      echo -n "threads=$t mode=$m chunk=$c "
      STITCH_B200_COPY_THREADS=$t STITCH_B200_STAGE_MODE=$m STITCH_B200_STAGE_CHUNK_MB=$c timeout 300 python scripts/sync_breakdown.py 40 2>&1 | tail -1
    done
  done
done

# K2: bulk-async tiles (k_stage_apply_bulk) vs per-warp window copies (k_stage_apply_std),
# device time from a captured graph of 50 applies
for c in 2 3; do
  for v in "" "IRK_NO_BULK=1"; do
    echo "== config $c $v"
    env $v timeout 300 python profiles/micro_stage.py $c 2>&1 | tail -4
  done
done

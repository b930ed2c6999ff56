# A/B of the chains' grid sizes (CTAs per SM, WS_GRID_*) on BJ configs[1]: step time of each setting
for setting in "" "WS_GRID_ROWS=4" "WS_GRID_ROWS=3" "WS_GRID_WARP=4" "WS_GRID_WARP=3" "WS_GRID_SCLASS=8" "WS_GRID_CPLANES=4" \
    "WS_GRID_ROWS=4 WS_GRID_WARP=4" "WS_GRID_ROWS=4 WS_GRID_WARP=3 WS_GRID_SCLASS=8 WS_GRID_CPLANES=4" \
    "WS_GRID_ROWS=6 WS_GRID_WARP=4 WS_GRID_CPLANES=4" "WS_GRID_SMSET=4" "WS_GRID_FOLD=3"; do
  for i in 1 2; do
    echo "[$setting] $(env $setting python scripts/probe.py configs1 2>&1 | head -1)"
  done
done

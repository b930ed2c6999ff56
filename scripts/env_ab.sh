# A/B of run-time switches on BJ configs[1] (probe: estimate only) and the headline bench step
for setting in "" "WS_ROWMAIN=0" "WS_PDL=0" "WS_ROWMAIN=0 WS_PDL=0"; do
  for i in 1 2; do
    echo "[$setting] $(env $setting python scripts/probe.py configs1 2>&1 | head -1)"
  done
done

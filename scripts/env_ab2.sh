# A/B of run-time switches on BJ configs[1] and LBM15 (probe: estimate only, graph replay)
for setting in "" "WS_PRIO=1" "WS_PRIO=2" "" "WS_PRIO=1" "WS_PRIO=2"; do
  echo "[$setting] $(env $setting python scripts/probe.py configs1 2>&1 | head -1)"
  echo "[$setting] $(env $setting python scripts/probe.py lbm15 2>&1 | head -1)"
done

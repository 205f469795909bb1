#!/bin/bash
# A/B the simulated p = 8 peer reduce kernel of several builds (ncu launch durations): bash scripts/ab_peer.sh lib...
for L in "$@"; do
  echo -n "$(basename $L) "
  APS_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/peer_sim.py 8 3 2>/dev/null \
    | grep peer_reduce | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' '
  echo
done

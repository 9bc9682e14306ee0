#!/bin/bash
# A/B per-launch device times of one MVM for several library builds / env settings:
#   tools/ab_launch.sh CONFIG REPS lib1.so[,VAR=val,...] lib2.so ...
cfg=$1; reps=$2; shift 2
for i in $(seq 1 $reps); do
  for spec in "$@"; do
    IFS=',' read -r lib envs <<< "$spec"
    echo -n "$(basename $lib) $envs: "
    env TSK_LIB=$PWD/$lib ${envs//,/ } timeout 300 python tools/launch_times.py $cfg 2>&1 | tail -n 1
  done
done

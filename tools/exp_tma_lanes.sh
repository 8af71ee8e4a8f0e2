#!/bin/bash
# register-staged vs TMA Schur update (QPB200_TC_TMA) at one lane / default lanes
for cfg in 4 5; do
  bash tools/exp_env.sh $cfg - QPB200_TC_TMA=42 QPB200_BLANES=1 "QPB200_BLANES=1 QPB200_TC_TMA=42"
done

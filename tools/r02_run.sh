#!/bin/bash
# round 2: GPU tests + config-5 bench of HEAD, then the config 3/4 convergence sweep
TAG=$1
bash tools/r02_check.sh $TAG
bash tools/r02_sweep2.sh

#!/bin/bash
# multicast availability on the box (NVLS needs the fabric manager on NVSwitch systems)
nvidia-smi -q | grep -iE -A3 "fabric|nvlink" | head -30
ls /dev | grep -i nvidia
ps aux | grep -i fabric | grep -v grep | head
python tests/helpers/nccl_world1.py 2>&1 | tail -2

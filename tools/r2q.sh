#!/bin/bash
O=gpurun_out; mkdir -p $O
TA=1 python tools/steps_probe.py sbm > $O/r2q_sbm_torch.txt 2>&1
TA=0 python tools/steps_probe.py sbm > $O/r2q_sbm_pool.txt 2>&1
TA=1 python tools/steps_probe.py cooc > $O/r2q_cooc_torch.txt 2>&1
echo done

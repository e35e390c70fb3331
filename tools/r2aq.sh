#!/bin/bash
O=gpurun_out; mkdir -p $O
bash tools/variants.sh "cur:" "acc1:LV_HUB_ACC_CTAS=1" "fin1:LV_HUB_FIN_CTAS=1" "fin2:LV_HUB_FIN_CTAS=2" "fin4:LV_HUB_FIN_CTAS=4" "cur2:" > $O/r2aq_variants.txt 2>&1
echo done

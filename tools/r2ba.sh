#!/bin/bash
O=gpurun_out; mkdir -p $O
rm -f $O/*.ncu-rep
bash tools/variants.sh "cur:" "w2u2:LV_TAB_W7=1" "w2u4:LV_TAB_W7=2" "w8u1:LV_TAB_W7=3" "w4u1:LV_TAB_W7=4" "cur2:" > $O/r2ba_variants.txt 2>&1
echo done

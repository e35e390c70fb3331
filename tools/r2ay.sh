#!/bin/bash
O=gpurun_out; mkdir -p $O
bash tools/variants.sh "cur:" "hu4:LV_SO=paper_1805_10904_b200/csrc/liblouvain_hu4.so" "hu2:LV_SO=paper_1805_10904_b200/csrc/liblouvain_hu2.so" "cur2:" > $O/r2ay_variants.txt 2>&1
echo done

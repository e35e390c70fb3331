#!/bin/bash
O=gpurun_out; mkdir -p $O
bash tools/variants.sh "cur:" "mb5:LV_SO=paper_1805_10904_b200/csrc/liblouvain_mb5.so" "mb6:LV_SO=paper_1805_10904_b200/csrc/liblouvain_mb6.so" "cur2:" "mb5b:LV_SO=paper_1805_10904_b200/csrc/liblouvain_mb5.so" > $O/r2ah_variants.txt 2>&1
echo done

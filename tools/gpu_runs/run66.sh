# 256-row work claims at d = 32 (half the table-head copies per row): A/B on C4 and C3
bash tools/qv.sh "ck256 base" "c4"
bash tools/qv.sh "ck256" "c3"

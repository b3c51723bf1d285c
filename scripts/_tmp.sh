A="--tables 1 --rows 10000000 --d 128 --pool-max 32 --pool-fixed --batch 32768 --zipf --bwd"
python scripts/emb_one.py $A > /dev/null && ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/emb_one.py $A --reps 1 > gpurun_out/zb.csv 2>/dev/null

python scripts/emb_one.py --tables 1 --rows 1000000 --d 64 --pool-max 32 --pool-fixed --batch 32768 --bwd
ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/emb_one.py --tables 1 --rows 1000000 --d 64 --pool-max 32 --pool-fixed --batch 32768 --bwd --reps 1 > gpurun_out/bwd1.csv 2>/dev/null

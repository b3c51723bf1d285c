python scripts/emb_one.py --tables 26 --rows 1000000 --d 16 --pool-max 1 --pool-fixed --batch 2048 --bwd --apply
python scripts/emb_one.py --bwd --apply

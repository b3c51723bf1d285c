A="--tables 1 --rows 10000000 --d 64 --pool-max 32 --pool-fixed --batch 32768"
echo "u64 $(python scripts/emb_one.py $A)"
echo "z64 $(python scripts/emb_one.py $A --zipf)"
echo "c3 $(python scripts/emb_one.py)"
echo "z128 $(python scripts/emb_one.py --tables 1 --rows 10000000 --d 128 --pool-max 32 --pool-fixed --batch 32768 --zipf)"
echo "u128 $(python scripts/emb_one.py --tables 1 --rows 10000000 --d 128 --pool-max 32 --pool-fixed --batch 32768)"
echo "z256 $(python scripts/emb_one.py --tables 1 --rows 10000000 --d 256 --pool-max 32 --pool-fixed --batch 32768 --zipf)"
timeout 300 python -m pytest tests/test_gpu_emb.py -q 2>&1 | tail -1

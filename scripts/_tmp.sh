for n in base t512 t1024 t512b64 t512b48; do echo "== $n"; DLRM_B200_LIB=$PWD/scratch/lib_$n.so python scripts/interact_bench.py; done

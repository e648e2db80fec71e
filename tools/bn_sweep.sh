for bn in 128 64 32; do
 echo "BN=$bn"; CG_TC_BN=$bn timeout 120 python tools/bench_train.py --configs C4,C3 --iters 20 2>&1 | grep ms_per_iter | cut -c1-90
done

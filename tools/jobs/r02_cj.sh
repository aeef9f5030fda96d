for i in 1 2; do
for lib in libhbp.so libhbp_alt.so; do
HBP_LIB_PATH=$PWD/paper_2504_08860_b200/$lib timeout 600 python tools/ab_ticket.py --config cfg2 --runs "static" --rounds 3 --iters 10 2>&1 | tail -1 | cut -c1-120 | sed "s/^/$lib /"
done
done
for lib in libhbp.so libhbp_alt.so; do
HBP_LIB_PATH=$PWD/paper_2504_08860_b200/$lib timeout 600 python tools/ab_ticket.py --config H --runs "static" --rounds 3 --iters 10 2>&1 | tail -1 | cut -c1-120 | sed "s/^/$lib /"
HBP_LIB_PATH=$PWD/paper_2504_08860_b200/$lib timeout 600 python tools/ab_ticket.py --config cfg5 --runs "static" --rounds 3 --iters 6 2>&1 | tail -1 | cut -c1-120 | sed "s/^/$lib /"
done

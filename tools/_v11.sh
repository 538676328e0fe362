bash tools/w2cycle.sh v11 --full --ncu

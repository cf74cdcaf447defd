for sk in 0 1 2 3; do echo "skip=$sk"; CFTFT_DEBUG_SKIP=$sk bash tools/benchline.sh C5 C2; done

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2203_08680_b200
timeout 1500 python tools/ab.py --rounds 2 --gens 300 base "keeploop:GOMIX_LIB=$L/libgomix_b200_keeploop.so" "nowalk:GOMIX_LIB=$L/libgomix_b200_nowalk.so" "both:GOMIX_LIB=$L/libgomix_b200_both.so" "head:GOMIX_LIB=$L/libgomix_b200_head.so" > gpurun_out/ab5.log 2>&1
grep round gpurun_out/ab5.log

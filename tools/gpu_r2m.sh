cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c3 c5_16 c5_1024 c5_4096; do
  GOMIX_LIB=paper_2203_08680_b200/libgomix_b200_probes.so timeout 300 python tools/prof_timeline.py $c > gpurun_out/r2m_timeline_$c.txt 2>&1
done

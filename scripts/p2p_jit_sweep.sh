# P2P occupancy / unroll sweep through BFMM_JIT_OPTS (NVRTC -D options); results in profiles/r01_p2p_flops.txt
for o in "" "-DBFMM_P2P_MINB=5" "-DBFMM_P2P_MINB=6" "-DBFMM_P2P_UNROLL=6 -DBFMM_P2P_MINB=5" "-DBFMM_P2P_UNROLL=4 -DBFMM_P2P_MINB=6" "-DBFMM_P2P_UNROLL=4 -DBFMM_P2P_MINB=8" "-DBFMM_P2P_UNROLL=12"; do
  echo "opts [$o]: $(BFMM_JIT_OPTS="$o" timeout 120 python scripts/p2p_time.py 2>&1 | tail -1)"
done

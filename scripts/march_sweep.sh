# k_diffusion_march plan sweep at one grid: cells per thread S x occupancy x i-splits (env knobs).
G=${G:-768}
for s in 1 2 4 8; do for occ in 2 3 4; do for sp in 0 1 2 3 4; do
  out=$(SOLOMON_DIFF_S=$s SOLOMON_DIFF_OCC=$occ SOLOMON_DIFF_SPLITS=$sp timeout 120 python scripts/time_diffusion.py $G 20 2>/dev/null | tail -1)
  echo "G=$G S=$s occ=$occ splits=$sp $out"
done; done; done

# Single-step diffusion3d GLUPS with a knob on/off ($KNOB over $VALS), interleaved, per grid.
KNOB=${KNOB:-SOLOMON_DIFF_AUTOTUNE}
for rep in 1 2; do for g in ${GRIDS:-256 512 640 768 896 1024}; do for v in ${VALS:-1 0}; do
  echo "$KNOB=$v $(env $KNOB=$v timeout 120 python scripts/time_diffusion.py $g 20 2>/dev/null | tail -1)"
done; done; done

# Round-2 status call: round-end suite + smoke + bench, then the profiling pass.
TAG=${TAG:-r2b} bash tools/gpu_round.sh
TAG=${TAG:-r2b} bash tools/gpu_prof.sh

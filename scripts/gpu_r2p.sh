bash scripts/gpu_profile.sh r2b

bash tools/gpu_checkpoint.sh
bash tools/gpu_jitmap_ab.sh

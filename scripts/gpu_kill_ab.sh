bash scripts/gpu_dev_all.sh k12
bash scripts/gpu_variants_full.sh kq kw main kq kw main

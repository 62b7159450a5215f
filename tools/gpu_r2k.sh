bash tools/cfg1_minb_ab.sh
bash tools/pack_smem_ab.sh

# Round-2 batch: the cfg1 occupancy and sharded-pack shared-memory A/Bs.
bash tools/cfg1_minb_ab.sh
bash tools/pack_smem_ab.sh

bash tools/_ab_cfg.sh cfg3

bash tools/_ab.sh

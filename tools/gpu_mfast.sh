for mf in 1000 2 4; do
  echo "mfast>=$mf"
  for shp in "128 128 16 128" "256 256 8 128" "512 512 4 128"; do MPCG_TC3_MFAST=$mf timeout 300 python tools/conv_probe.py $shp --time; done
done

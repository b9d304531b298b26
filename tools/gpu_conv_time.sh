# executor conv layer: GEMM kernel time and eager run time, deferred eps on/off, ResNet-18 shapes
for shp in "64 64 32 128" "128 128 16 128" "256 256 8 128" "512 512 4 128"; do
  for d in 1 0; do MPCG_EPS_DEFER=$d timeout 300 python tools/conv_probe.py $shp --time; done
done

# 3-layer conv3x3 + ReLU + 2x2 maxpool, 2-D (configs[0] 2-D variant)
pipeline crp2d
buffer input dims 3x66x66 elem 4
buffer conv1_w dims 16x3x3x3 elem 4
stage conv1 dims co:16,y:64,x:64 reduce ci:3 flops 18
  in input map ci*1+1, y*1+3, x*1+3
  in conv1_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu2 dims c:16,y:64,x:64 flops 1
  in conv1 map c*1+1, y*1+1, x*1+1
stage pool3 dims c:16,y:32,x:32 flops 4 output
  in relu2 map c*1+1, y*2+2, x*2+2

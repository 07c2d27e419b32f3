# VGG-16 probe: 13 valid 3x3 convs + ReLU, 5 max-pools, GAP, 2 FC (T=34)
pipeline vgg16
buffer input dims 3x252x252 elem 4
buffer conv1_w dims 64x3x3x3 elem 4
buffer conv3_w dims 64x64x3x3 elem 4
buffer conv6_w dims 128x64x3x3 elem 4
buffer conv8_w dims 128x128x3x3 elem 4
buffer conv11_w dims 256x128x3x3 elem 4
buffer conv13_w dims 256x256x3x3 elem 4
buffer conv15_w dims 256x256x3x3 elem 4
buffer conv18_w dims 512x256x3x3 elem 4
buffer conv20_w dims 512x512x3x3 elem 4
buffer conv22_w dims 512x512x3x3 elem 4
buffer conv25_w dims 512x512x3x3 elem 4
buffer conv27_w dims 512x512x3x3 elem 4
buffer conv29_w dims 512x512x3x3 elem 4
buffer fc33_w dims 4096x512 elem 4
buffer fc34_w dims 1000x4096 elem 4
stage conv1 dims co:64,y:250,x:250 reduce ci:3 flops 18
  in input map ci*1+1, y*1+3, x*1+3
  in conv1_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu2 dims c:64,y:250,x:250 flops 1
  in conv1 map c*1+1, y*1+1, x*1+1
stage conv3 dims co:64,y:248,x:248 reduce ci:64 flops 18
  in relu2 map ci*1+1, y*1+3, x*1+3
  in conv3_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu4 dims c:64,y:248,x:248 flops 1
  in conv3 map c*1+1, y*1+1, x*1+1
stage pool5 dims c:64,y:124,x:124 flops 4
  in relu4 map c*1+1, y*2+2, x*2+2
stage conv6 dims co:128,y:122,x:122 reduce ci:64 flops 18
  in pool5 map ci*1+1, y*1+3, x*1+3
  in conv6_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu7 dims c:128,y:122,x:122 flops 1
  in conv6 map c*1+1, y*1+1, x*1+1
stage conv8 dims co:128,y:120,x:120 reduce ci:128 flops 18
  in relu7 map ci*1+1, y*1+3, x*1+3
  in conv8_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu9 dims c:128,y:120,x:120 flops 1
  in conv8 map c*1+1, y*1+1, x*1+1
stage pool10 dims c:128,y:60,x:60 flops 4
  in relu9 map c*1+1, y*2+2, x*2+2
stage conv11 dims co:256,y:58,x:58 reduce ci:128 flops 18
  in pool10 map ci*1+1, y*1+3, x*1+3
  in conv11_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu12 dims c:256,y:58,x:58 flops 1
  in conv11 map c*1+1, y*1+1, x*1+1
stage conv13 dims co:256,y:56,x:56 reduce ci:256 flops 18
  in relu12 map ci*1+1, y*1+3, x*1+3
  in conv13_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu14 dims c:256,y:56,x:56 flops 1
  in conv13 map c*1+1, y*1+1, x*1+1
stage conv15 dims co:256,y:54,x:54 reduce ci:256 flops 18
  in relu14 map ci*1+1, y*1+3, x*1+3
  in conv15_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu16 dims c:256,y:54,x:54 flops 1
  in conv15 map c*1+1, y*1+1, x*1+1
stage pool17 dims c:256,y:27,x:27 flops 4
  in relu16 map c*1+1, y*2+2, x*2+2
stage conv18 dims co:512,y:25,x:25 reduce ci:256 flops 18
  in pool17 map ci*1+1, y*1+3, x*1+3
  in conv18_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu19 dims c:512,y:25,x:25 flops 1
  in conv18 map c*1+1, y*1+1, x*1+1
stage conv20 dims co:512,y:23,x:23 reduce ci:512 flops 18
  in relu19 map ci*1+1, y*1+3, x*1+3
  in conv20_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu21 dims c:512,y:23,x:23 flops 1
  in conv20 map c*1+1, y*1+1, x*1+1
stage conv22 dims co:512,y:21,x:21 reduce ci:512 flops 18
  in relu21 map ci*1+1, y*1+3, x*1+3
  in conv22_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu23 dims c:512,y:21,x:21 flops 1
  in conv22 map c*1+1, y*1+1, x*1+1
stage pool24 dims c:512,y:10,x:10 flops 4
  in relu23 map c*1+1, y*2+2, x*2+2
stage conv25 dims co:512,y:8,x:8 reduce ci:512 flops 18
  in pool24 map ci*1+1, y*1+3, x*1+3
  in conv25_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu26 dims c:512,y:8,x:8 flops 1
  in conv25 map c*1+1, y*1+1, x*1+1
stage conv27 dims co:512,y:6,x:6 reduce ci:512 flops 18
  in relu26 map ci*1+1, y*1+3, x*1+3
  in conv27_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu28 dims c:512,y:6,x:6 flops 1
  in conv27 map c*1+1, y*1+1, x*1+1
stage conv29 dims co:512,y:4,x:4 reduce ci:512 flops 18
  in relu28 map ci*1+1, y*1+3, x*1+3
  in conv29_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu30 dims c:512,y:4,x:4 flops 1
  in conv29 map c*1+1, y*1+1, x*1+1
stage pool31 dims c:512,y:2,x:2 flops 4
  in relu30 map c*1+1, y*2+2, x*2+2
stage gap32 dims c:512 reduce y:2,x:2 flops 1
  in pool31 map c*1+1, y*1+1, x*1+1
stage fc33 dims o:4096 reduce i:512 flops 2
  in gap32 map i*1+1
  in fc33_w map o*1+1, i*1+1
stage fc34 dims o:1000 reduce i:4096 flops 2 output
  in fc33 map i*1+1
  in fc34_w map o*1+1, i*1+1

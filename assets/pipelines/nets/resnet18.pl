# ResNet-18 probe: valid convs, corner-cropped skips, GAP+FC (T=48)
pipeline resnet18
buffer input dims 3x544x544 elem 4
buffer conv1_w dims 64x3x7x7 elem 4
buffer conv4_w dims 64x64x3x3 elem 4
buffer conv6_w dims 64x64x3x3 elem 4
buffer conv9_w dims 64x64x3x3 elem 4
buffer conv11_w dims 64x64x3x3 elem 4
buffer conv14_w dims 128x64x3x3 elem 4
buffer conv16_w dims 128x128x3x3 elem 4
buffer proj17_w dims 128x64x1x1 elem 4
buffer conv20_w dims 128x128x3x3 elem 4
buffer conv22_w dims 128x128x3x3 elem 4
buffer conv25_w dims 256x128x3x3 elem 4
buffer conv27_w dims 256x256x3x3 elem 4
buffer proj28_w dims 256x128x1x1 elem 4
buffer conv31_w dims 256x256x3x3 elem 4
buffer conv33_w dims 256x256x3x3 elem 4
buffer conv36_w dims 512x256x3x3 elem 4
buffer conv38_w dims 512x512x3x3 elem 4
buffer proj39_w dims 512x256x1x1 elem 4
buffer conv42_w dims 512x512x3x3 elem 4
buffer conv44_w dims 512x512x3x3 elem 4
buffer fc48_w dims 1000x512 elem 4
stage conv1 dims co:64,y:269,x:269 reduce ci:3 flops 98
  in input map ci*1+1, y*2+7, x*2+7
  in conv1_w map co*1+1, ci*1+1, _*0+7, _*0+7
stage relu2 dims c:64,y:269,x:269 flops 1
  in conv1 map c*1+1, y*1+1, x*1+1
stage pool3 dims c:64,y:134,x:134 flops 9
  in relu2 map c*1+1, y*2+3, x*2+3
stage conv4 dims co:64,y:132,x:132 reduce ci:64 flops 18
  in pool3 map ci*1+1, y*1+3, x*1+3
  in conv4_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu5 dims c:64,y:132,x:132 flops 1
  in conv4 map c*1+1, y*1+1, x*1+1
stage conv6 dims co:64,y:130,x:130 reduce ci:64 flops 18
  in relu5 map ci*1+1, y*1+3, x*1+3
  in conv6_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage add7 dims c:64,y:130,x:130 flops 1
  in conv6 map c*1+1, y*1+1, x*1+1
  in pool3 map c*1+1, y*1+1, x*1+1
stage relu8 dims c:64,y:130,x:130 flops 1
  in add7 map c*1+1, y*1+1, x*1+1
stage conv9 dims co:64,y:128,x:128 reduce ci:64 flops 18
  in relu8 map ci*1+1, y*1+3, x*1+3
  in conv9_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu10 dims c:64,y:128,x:128 flops 1
  in conv9 map c*1+1, y*1+1, x*1+1
stage conv11 dims co:64,y:126,x:126 reduce ci:64 flops 18
  in relu10 map ci*1+1, y*1+3, x*1+3
  in conv11_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage add12 dims c:64,y:126,x:126 flops 1
  in conv11 map c*1+1, y*1+1, x*1+1
  in relu8 map c*1+1, y*1+1, x*1+1
stage relu13 dims c:64,y:126,x:126 flops 1
  in add12 map c*1+1, y*1+1, x*1+1
stage conv14 dims co:128,y:62,x:62 reduce ci:64 flops 18
  in relu13 map ci*1+1, y*2+3, x*2+3
  in conv14_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu15 dims c:128,y:62,x:62 flops 1
  in conv14 map c*1+1, y*1+1, x*1+1
stage conv16 dims co:128,y:60,x:60 reduce ci:128 flops 18
  in relu15 map ci*1+1, y*1+3, x*1+3
  in conv16_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage proj17 dims co:128,y:63,x:63 reduce ci:64 flops 2
  in relu13 map ci*1+1, y*2+1, x*2+1
  in proj17_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add18 dims c:128,y:60,x:60 flops 1
  in conv16 map c*1+1, y*1+1, x*1+1
  in proj17 map c*1+1, y*1+1, x*1+1
stage relu19 dims c:128,y:60,x:60 flops 1
  in add18 map c*1+1, y*1+1, x*1+1
stage conv20 dims co:128,y:58,x:58 reduce ci:128 flops 18
  in relu19 map ci*1+1, y*1+3, x*1+3
  in conv20_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu21 dims c:128,y:58,x:58 flops 1
  in conv20 map c*1+1, y*1+1, x*1+1
stage conv22 dims co:128,y:56,x:56 reduce ci:128 flops 18
  in relu21 map ci*1+1, y*1+3, x*1+3
  in conv22_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage add23 dims c:128,y:56,x:56 flops 1
  in conv22 map c*1+1, y*1+1, x*1+1
  in relu19 map c*1+1, y*1+1, x*1+1
stage relu24 dims c:128,y:56,x:56 flops 1
  in add23 map c*1+1, y*1+1, x*1+1
stage conv25 dims co:256,y:27,x:27 reduce ci:128 flops 18
  in relu24 map ci*1+1, y*2+3, x*2+3
  in conv25_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu26 dims c:256,y:27,x:27 flops 1
  in conv25 map c*1+1, y*1+1, x*1+1
stage conv27 dims co:256,y:25,x:25 reduce ci:256 flops 18
  in relu26 map ci*1+1, y*1+3, x*1+3
  in conv27_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage proj28 dims co:256,y:28,x:28 reduce ci:128 flops 2
  in relu24 map ci*1+1, y*2+1, x*2+1
  in proj28_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add29 dims c:256,y:25,x:25 flops 1
  in conv27 map c*1+1, y*1+1, x*1+1
  in proj28 map c*1+1, y*1+1, x*1+1
stage relu30 dims c:256,y:25,x:25 flops 1
  in add29 map c*1+1, y*1+1, x*1+1
stage conv31 dims co:256,y:23,x:23 reduce ci:256 flops 18
  in relu30 map ci*1+1, y*1+3, x*1+3
  in conv31_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu32 dims c:256,y:23,x:23 flops 1
  in conv31 map c*1+1, y*1+1, x*1+1
stage conv33 dims co:256,y:21,x:21 reduce ci:256 flops 18
  in relu32 map ci*1+1, y*1+3, x*1+3
  in conv33_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage add34 dims c:256,y:21,x:21 flops 1
  in conv33 map c*1+1, y*1+1, x*1+1
  in relu30 map c*1+1, y*1+1, x*1+1
stage relu35 dims c:256,y:21,x:21 flops 1
  in add34 map c*1+1, y*1+1, x*1+1
stage conv36 dims co:512,y:10,x:10 reduce ci:256 flops 18
  in relu35 map ci*1+1, y*2+3, x*2+3
  in conv36_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu37 dims c:512,y:10,x:10 flops 1
  in conv36 map c*1+1, y*1+1, x*1+1
stage conv38 dims co:512,y:8,x:8 reduce ci:512 flops 18
  in relu37 map ci*1+1, y*1+3, x*1+3
  in conv38_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage proj39 dims co:512,y:11,x:11 reduce ci:256 flops 2
  in relu35 map ci*1+1, y*2+1, x*2+1
  in proj39_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add40 dims c:512,y:8,x:8 flops 1
  in conv38 map c*1+1, y*1+1, x*1+1
  in proj39 map c*1+1, y*1+1, x*1+1
stage relu41 dims c:512,y:8,x:8 flops 1
  in add40 map c*1+1, y*1+1, x*1+1
stage conv42 dims co:512,y:6,x:6 reduce ci:512 flops 18
  in relu41 map ci*1+1, y*1+3, x*1+3
  in conv42_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu43 dims c:512,y:6,x:6 flops 1
  in conv42 map c*1+1, y*1+1, x*1+1
stage conv44 dims co:512,y:4,x:4 reduce ci:512 flops 18
  in relu43 map ci*1+1, y*1+3, x*1+3
  in conv44_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage add45 dims c:512,y:4,x:4 flops 1
  in conv44 map c*1+1, y*1+1, x*1+1
  in relu41 map c*1+1, y*1+1, x*1+1
stage relu46 dims c:512,y:4,x:4 flops 1
  in add45 map c*1+1, y*1+1, x*1+1
stage gap47 dims c:512 reduce y:4,x:4 flops 1
  in relu46 map c*1+1, y*1+1, x*1+1
stage fc48 dims o:1000 reduce i:512 flops 2 output
  in gap47 map i*1+1
  in fc48_w map o*1+1, i*1+1

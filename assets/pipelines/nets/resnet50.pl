# ResNet-50 probe: bottleneck blocks, valid convs, GAP+FC (T=121)
pipeline resnet50
buffer input dims 3x544x544 elem 4
buffer conv1_w dims 64x3x7x7 elem 4
buffer conv4_w dims 64x64x1x1 elem 4
buffer conv6_w dims 64x64x3x3 elem 4
buffer conv8_w dims 256x64x1x1 elem 4
buffer proj9_w dims 256x64x1x1 elem 4
buffer conv12_w dims 64x256x1x1 elem 4
buffer conv14_w dims 64x64x3x3 elem 4
buffer conv16_w dims 256x64x1x1 elem 4
buffer conv19_w dims 64x256x1x1 elem 4
buffer conv21_w dims 64x64x3x3 elem 4
buffer conv23_w dims 256x64x1x1 elem 4
buffer conv26_w dims 128x256x1x1 elem 4
buffer conv28_w dims 128x128x3x3 elem 4
buffer conv30_w dims 512x128x1x1 elem 4
buffer proj31_w dims 512x256x1x1 elem 4
buffer conv34_w dims 128x512x1x1 elem 4
buffer conv36_w dims 128x128x3x3 elem 4
buffer conv38_w dims 512x128x1x1 elem 4
buffer conv41_w dims 128x512x1x1 elem 4
buffer conv43_w dims 128x128x3x3 elem 4
buffer conv45_w dims 512x128x1x1 elem 4
buffer conv48_w dims 128x512x1x1 elem 4
buffer conv50_w dims 128x128x3x3 elem 4
buffer conv52_w dims 512x128x1x1 elem 4
buffer conv55_w dims 256x512x1x1 elem 4
buffer conv57_w dims 256x256x3x3 elem 4
buffer conv59_w dims 1024x256x1x1 elem 4
buffer proj60_w dims 1024x512x1x1 elem 4
buffer conv63_w dims 256x1024x1x1 elem 4
buffer conv65_w dims 256x256x3x3 elem 4
buffer conv67_w dims 1024x256x1x1 elem 4
buffer conv70_w dims 256x1024x1x1 elem 4
buffer conv72_w dims 256x256x3x3 elem 4
buffer conv74_w dims 1024x256x1x1 elem 4
buffer conv77_w dims 256x1024x1x1 elem 4
buffer conv79_w dims 256x256x3x3 elem 4
buffer conv81_w dims 1024x256x1x1 elem 4
buffer conv84_w dims 256x1024x1x1 elem 4
buffer conv86_w dims 256x256x3x3 elem 4
buffer conv88_w dims 1024x256x1x1 elem 4
buffer conv91_w dims 256x1024x1x1 elem 4
buffer conv93_w dims 256x256x3x3 elem 4
buffer conv95_w dims 1024x256x1x1 elem 4
buffer conv98_w dims 512x1024x1x1 elem 4
buffer conv100_w dims 512x512x3x3 elem 4
buffer conv102_w dims 2048x512x1x1 elem 4
buffer proj103_w dims 2048x1024x1x1 elem 4
buffer conv106_w dims 512x2048x1x1 elem 4
buffer conv108_w dims 512x512x3x3 elem 4
buffer conv110_w dims 2048x512x1x1 elem 4
buffer conv113_w dims 512x2048x1x1 elem 4
buffer conv115_w dims 512x512x3x3 elem 4
buffer conv117_w dims 2048x512x1x1 elem 4
buffer fc121_w dims 1000x2048 elem 4
stage conv1 dims co:64,y:269,x:269 reduce ci:3 flops 98
  in input map ci*1+1, y*2+7, x*2+7
  in conv1_w map co*1+1, ci*1+1, _*0+7, _*0+7
stage relu2 dims c:64,y:269,x:269 flops 1
  in conv1 map c*1+1, y*1+1, x*1+1
stage pool3 dims c:64,y:134,x:134 flops 9
  in relu2 map c*1+1, y*2+3, x*2+3
stage conv4 dims co:64,y:134,x:134 reduce ci:64 flops 2
  in pool3 map ci*1+1, y*1+1, x*1+1
  in conv4_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu5 dims c:64,y:134,x:134 flops 1
  in conv4 map c*1+1, y*1+1, x*1+1
stage conv6 dims co:64,y:132,x:132 reduce ci:64 flops 18
  in relu5 map ci*1+1, y*1+3, x*1+3
  in conv6_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu7 dims c:64,y:132,x:132 flops 1
  in conv6 map c*1+1, y*1+1, x*1+1
stage conv8 dims co:256,y:132,x:132 reduce ci:64 flops 2
  in relu7 map ci*1+1, y*1+1, x*1+1
  in conv8_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage proj9 dims co:256,y:134,x:134 reduce ci:64 flops 2
  in pool3 map ci*1+1, y*1+1, x*1+1
  in proj9_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add10 dims c:256,y:132,x:132 flops 1
  in conv8 map c*1+1, y*1+1, x*1+1
  in proj9 map c*1+1, y*1+1, x*1+1
stage relu11 dims c:256,y:132,x:132 flops 1
  in add10 map c*1+1, y*1+1, x*1+1
stage conv12 dims co:64,y:132,x:132 reduce ci:256 flops 2
  in relu11 map ci*1+1, y*1+1, x*1+1
  in conv12_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu13 dims c:64,y:132,x:132 flops 1
  in conv12 map c*1+1, y*1+1, x*1+1
stage conv14 dims co:64,y:130,x:130 reduce ci:64 flops 18
  in relu13 map ci*1+1, y*1+3, x*1+3
  in conv14_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu15 dims c:64,y:130,x:130 flops 1
  in conv14 map c*1+1, y*1+1, x*1+1
stage conv16 dims co:256,y:130,x:130 reduce ci:64 flops 2
  in relu15 map ci*1+1, y*1+1, x*1+1
  in conv16_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add17 dims c:256,y:130,x:130 flops 1
  in conv16 map c*1+1, y*1+1, x*1+1
  in relu11 map c*1+1, y*1+1, x*1+1
stage relu18 dims c:256,y:130,x:130 flops 1
  in add17 map c*1+1, y*1+1, x*1+1
stage conv19 dims co:64,y:130,x:130 reduce ci:256 flops 2
  in relu18 map ci*1+1, y*1+1, x*1+1
  in conv19_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu20 dims c:64,y:130,x:130 flops 1
  in conv19 map c*1+1, y*1+1, x*1+1
stage conv21 dims co:64,y:128,x:128 reduce ci:64 flops 18
  in relu20 map ci*1+1, y*1+3, x*1+3
  in conv21_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu22 dims c:64,y:128,x:128 flops 1
  in conv21 map c*1+1, y*1+1, x*1+1
stage conv23 dims co:256,y:128,x:128 reduce ci:64 flops 2
  in relu22 map ci*1+1, y*1+1, x*1+1
  in conv23_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add24 dims c:256,y:128,x:128 flops 1
  in conv23 map c*1+1, y*1+1, x*1+1
  in relu18 map c*1+1, y*1+1, x*1+1
stage relu25 dims c:256,y:128,x:128 flops 1
  in add24 map c*1+1, y*1+1, x*1+1
stage conv26 dims co:128,y:128,x:128 reduce ci:256 flops 2
  in relu25 map ci*1+1, y*1+1, x*1+1
  in conv26_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu27 dims c:128,y:128,x:128 flops 1
  in conv26 map c*1+1, y*1+1, x*1+1
stage conv28 dims co:128,y:63,x:63 reduce ci:128 flops 18
  in relu27 map ci*1+1, y*2+3, x*2+3
  in conv28_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu29 dims c:128,y:63,x:63 flops 1
  in conv28 map c*1+1, y*1+1, x*1+1
stage conv30 dims co:512,y:63,x:63 reduce ci:128 flops 2
  in relu29 map ci*1+1, y*1+1, x*1+1
  in conv30_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage proj31 dims co:512,y:64,x:64 reduce ci:256 flops 2
  in relu25 map ci*1+1, y*2+1, x*2+1
  in proj31_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add32 dims c:512,y:63,x:63 flops 1
  in conv30 map c*1+1, y*1+1, x*1+1
  in proj31 map c*1+1, y*1+1, x*1+1
stage relu33 dims c:512,y:63,x:63 flops 1
  in add32 map c*1+1, y*1+1, x*1+1
stage conv34 dims co:128,y:63,x:63 reduce ci:512 flops 2
  in relu33 map ci*1+1, y*1+1, x*1+1
  in conv34_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu35 dims c:128,y:63,x:63 flops 1
  in conv34 map c*1+1, y*1+1, x*1+1
stage conv36 dims co:128,y:61,x:61 reduce ci:128 flops 18
  in relu35 map ci*1+1, y*1+3, x*1+3
  in conv36_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu37 dims c:128,y:61,x:61 flops 1
  in conv36 map c*1+1, y*1+1, x*1+1
stage conv38 dims co:512,y:61,x:61 reduce ci:128 flops 2
  in relu37 map ci*1+1, y*1+1, x*1+1
  in conv38_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add39 dims c:512,y:61,x:61 flops 1
  in conv38 map c*1+1, y*1+1, x*1+1
  in relu33 map c*1+1, y*1+1, x*1+1
stage relu40 dims c:512,y:61,x:61 flops 1
  in add39 map c*1+1, y*1+1, x*1+1
stage conv41 dims co:128,y:61,x:61 reduce ci:512 flops 2
  in relu40 map ci*1+1, y*1+1, x*1+1
  in conv41_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu42 dims c:128,y:61,x:61 flops 1
  in conv41 map c*1+1, y*1+1, x*1+1
stage conv43 dims co:128,y:59,x:59 reduce ci:128 flops 18
  in relu42 map ci*1+1, y*1+3, x*1+3
  in conv43_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu44 dims c:128,y:59,x:59 flops 1
  in conv43 map c*1+1, y*1+1, x*1+1
stage conv45 dims co:512,y:59,x:59 reduce ci:128 flops 2
  in relu44 map ci*1+1, y*1+1, x*1+1
  in conv45_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add46 dims c:512,y:59,x:59 flops 1
  in conv45 map c*1+1, y*1+1, x*1+1
  in relu40 map c*1+1, y*1+1, x*1+1
stage relu47 dims c:512,y:59,x:59 flops 1
  in add46 map c*1+1, y*1+1, x*1+1
stage conv48 dims co:128,y:59,x:59 reduce ci:512 flops 2
  in relu47 map ci*1+1, y*1+1, x*1+1
  in conv48_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu49 dims c:128,y:59,x:59 flops 1
  in conv48 map c*1+1, y*1+1, x*1+1
stage conv50 dims co:128,y:57,x:57 reduce ci:128 flops 18
  in relu49 map ci*1+1, y*1+3, x*1+3
  in conv50_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu51 dims c:128,y:57,x:57 flops 1
  in conv50 map c*1+1, y*1+1, x*1+1
stage conv52 dims co:512,y:57,x:57 reduce ci:128 flops 2
  in relu51 map ci*1+1, y*1+1, x*1+1
  in conv52_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add53 dims c:512,y:57,x:57 flops 1
  in conv52 map c*1+1, y*1+1, x*1+1
  in relu47 map c*1+1, y*1+1, x*1+1
stage relu54 dims c:512,y:57,x:57 flops 1
  in add53 map c*1+1, y*1+1, x*1+1
stage conv55 dims co:256,y:57,x:57 reduce ci:512 flops 2
  in relu54 map ci*1+1, y*1+1, x*1+1
  in conv55_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu56 dims c:256,y:57,x:57 flops 1
  in conv55 map c*1+1, y*1+1, x*1+1
stage conv57 dims co:256,y:28,x:28 reduce ci:256 flops 18
  in relu56 map ci*1+1, y*2+3, x*2+3
  in conv57_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu58 dims c:256,y:28,x:28 flops 1
  in conv57 map c*1+1, y*1+1, x*1+1
stage conv59 dims co:1024,y:28,x:28 reduce ci:256 flops 2
  in relu58 map ci*1+1, y*1+1, x*1+1
  in conv59_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage proj60 dims co:1024,y:29,x:29 reduce ci:512 flops 2
  in relu54 map ci*1+1, y*2+1, x*2+1
  in proj60_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add61 dims c:1024,y:28,x:28 flops 1
  in conv59 map c*1+1, y*1+1, x*1+1
  in proj60 map c*1+1, y*1+1, x*1+1
stage relu62 dims c:1024,y:28,x:28 flops 1
  in add61 map c*1+1, y*1+1, x*1+1
stage conv63 dims co:256,y:28,x:28 reduce ci:1024 flops 2
  in relu62 map ci*1+1, y*1+1, x*1+1
  in conv63_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu64 dims c:256,y:28,x:28 flops 1
  in conv63 map c*1+1, y*1+1, x*1+1
stage conv65 dims co:256,y:26,x:26 reduce ci:256 flops 18
  in relu64 map ci*1+1, y*1+3, x*1+3
  in conv65_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu66 dims c:256,y:26,x:26 flops 1
  in conv65 map c*1+1, y*1+1, x*1+1
stage conv67 dims co:1024,y:26,x:26 reduce ci:256 flops 2
  in relu66 map ci*1+1, y*1+1, x*1+1
  in conv67_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add68 dims c:1024,y:26,x:26 flops 1
  in conv67 map c*1+1, y*1+1, x*1+1
  in relu62 map c*1+1, y*1+1, x*1+1
stage relu69 dims c:1024,y:26,x:26 flops 1
  in add68 map c*1+1, y*1+1, x*1+1
stage conv70 dims co:256,y:26,x:26 reduce ci:1024 flops 2
  in relu69 map ci*1+1, y*1+1, x*1+1
  in conv70_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu71 dims c:256,y:26,x:26 flops 1
  in conv70 map c*1+1, y*1+1, x*1+1
stage conv72 dims co:256,y:24,x:24 reduce ci:256 flops 18
  in relu71 map ci*1+1, y*1+3, x*1+3
  in conv72_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu73 dims c:256,y:24,x:24 flops 1
  in conv72 map c*1+1, y*1+1, x*1+1
stage conv74 dims co:1024,y:24,x:24 reduce ci:256 flops 2
  in relu73 map ci*1+1, y*1+1, x*1+1
  in conv74_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add75 dims c:1024,y:24,x:24 flops 1
  in conv74 map c*1+1, y*1+1, x*1+1
  in relu69 map c*1+1, y*1+1, x*1+1
stage relu76 dims c:1024,y:24,x:24 flops 1
  in add75 map c*1+1, y*1+1, x*1+1
stage conv77 dims co:256,y:24,x:24 reduce ci:1024 flops 2
  in relu76 map ci*1+1, y*1+1, x*1+1
  in conv77_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu78 dims c:256,y:24,x:24 flops 1
  in conv77 map c*1+1, y*1+1, x*1+1
stage conv79 dims co:256,y:22,x:22 reduce ci:256 flops 18
  in relu78 map ci*1+1, y*1+3, x*1+3
  in conv79_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu80 dims c:256,y:22,x:22 flops 1
  in conv79 map c*1+1, y*1+1, x*1+1
stage conv81 dims co:1024,y:22,x:22 reduce ci:256 flops 2
  in relu80 map ci*1+1, y*1+1, x*1+1
  in conv81_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add82 dims c:1024,y:22,x:22 flops 1
  in conv81 map c*1+1, y*1+1, x*1+1
  in relu76 map c*1+1, y*1+1, x*1+1
stage relu83 dims c:1024,y:22,x:22 flops 1
  in add82 map c*1+1, y*1+1, x*1+1
stage conv84 dims co:256,y:22,x:22 reduce ci:1024 flops 2
  in relu83 map ci*1+1, y*1+1, x*1+1
  in conv84_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu85 dims c:256,y:22,x:22 flops 1
  in conv84 map c*1+1, y*1+1, x*1+1
stage conv86 dims co:256,y:20,x:20 reduce ci:256 flops 18
  in relu85 map ci*1+1, y*1+3, x*1+3
  in conv86_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu87 dims c:256,y:20,x:20 flops 1
  in conv86 map c*1+1, y*1+1, x*1+1
stage conv88 dims co:1024,y:20,x:20 reduce ci:256 flops 2
  in relu87 map ci*1+1, y*1+1, x*1+1
  in conv88_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add89 dims c:1024,y:20,x:20 flops 1
  in conv88 map c*1+1, y*1+1, x*1+1
  in relu83 map c*1+1, y*1+1, x*1+1
stage relu90 dims c:1024,y:20,x:20 flops 1
  in add89 map c*1+1, y*1+1, x*1+1
stage conv91 dims co:256,y:20,x:20 reduce ci:1024 flops 2
  in relu90 map ci*1+1, y*1+1, x*1+1
  in conv91_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu92 dims c:256,y:20,x:20 flops 1
  in conv91 map c*1+1, y*1+1, x*1+1
stage conv93 dims co:256,y:18,x:18 reduce ci:256 flops 18
  in relu92 map ci*1+1, y*1+3, x*1+3
  in conv93_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu94 dims c:256,y:18,x:18 flops 1
  in conv93 map c*1+1, y*1+1, x*1+1
stage conv95 dims co:1024,y:18,x:18 reduce ci:256 flops 2
  in relu94 map ci*1+1, y*1+1, x*1+1
  in conv95_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add96 dims c:1024,y:18,x:18 flops 1
  in conv95 map c*1+1, y*1+1, x*1+1
  in relu90 map c*1+1, y*1+1, x*1+1
stage relu97 dims c:1024,y:18,x:18 flops 1
  in add96 map c*1+1, y*1+1, x*1+1
stage conv98 dims co:512,y:18,x:18 reduce ci:1024 flops 2
  in relu97 map ci*1+1, y*1+1, x*1+1
  in conv98_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu99 dims c:512,y:18,x:18 flops 1
  in conv98 map c*1+1, y*1+1, x*1+1
stage conv100 dims co:512,y:8,x:8 reduce ci:512 flops 18
  in relu99 map ci*1+1, y*2+3, x*2+3
  in conv100_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu101 dims c:512,y:8,x:8 flops 1
  in conv100 map c*1+1, y*1+1, x*1+1
stage conv102 dims co:2048,y:8,x:8 reduce ci:512 flops 2
  in relu101 map ci*1+1, y*1+1, x*1+1
  in conv102_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage proj103 dims co:2048,y:9,x:9 reduce ci:1024 flops 2
  in relu97 map ci*1+1, y*2+1, x*2+1
  in proj103_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add104 dims c:2048,y:8,x:8 flops 1
  in conv102 map c*1+1, y*1+1, x*1+1
  in proj103 map c*1+1, y*1+1, x*1+1
stage relu105 dims c:2048,y:8,x:8 flops 1
  in add104 map c*1+1, y*1+1, x*1+1
stage conv106 dims co:512,y:8,x:8 reduce ci:2048 flops 2
  in relu105 map ci*1+1, y*1+1, x*1+1
  in conv106_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu107 dims c:512,y:8,x:8 flops 1
  in conv106 map c*1+1, y*1+1, x*1+1
stage conv108 dims co:512,y:6,x:6 reduce ci:512 flops 18
  in relu107 map ci*1+1, y*1+3, x*1+3
  in conv108_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu109 dims c:512,y:6,x:6 flops 1
  in conv108 map c*1+1, y*1+1, x*1+1
stage conv110 dims co:2048,y:6,x:6 reduce ci:512 flops 2
  in relu109 map ci*1+1, y*1+1, x*1+1
  in conv110_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add111 dims c:2048,y:6,x:6 flops 1
  in conv110 map c*1+1, y*1+1, x*1+1
  in relu105 map c*1+1, y*1+1, x*1+1
stage relu112 dims c:2048,y:6,x:6 flops 1
  in add111 map c*1+1, y*1+1, x*1+1
stage conv113 dims co:512,y:6,x:6 reduce ci:2048 flops 2
  in relu112 map ci*1+1, y*1+1, x*1+1
  in conv113_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu114 dims c:512,y:6,x:6 flops 1
  in conv113 map c*1+1, y*1+1, x*1+1
stage conv115 dims co:512,y:4,x:4 reduce ci:512 flops 18
  in relu114 map ci*1+1, y*1+3, x*1+3
  in conv115_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu116 dims c:512,y:4,x:4 flops 1
  in conv115 map c*1+1, y*1+1, x*1+1
stage conv117 dims co:2048,y:4,x:4 reduce ci:512 flops 2
  in relu116 map ci*1+1, y*1+1, x*1+1
  in conv117_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add118 dims c:2048,y:4,x:4 flops 1
  in conv117 map c*1+1, y*1+1, x*1+1
  in relu112 map c*1+1, y*1+1, x*1+1
stage relu119 dims c:2048,y:4,x:4 flops 1
  in add118 map c*1+1, y*1+1, x*1+1
stage gap120 dims c:2048 reduce y:4,x:4 flops 1
  in relu119 map c*1+1, y*1+1, x*1+1
stage fc121 dims o:1000 reduce i:2048 flops 2 output
  in gap120 map i*1+1
  in fc121_w map o*1+1, i*1+1

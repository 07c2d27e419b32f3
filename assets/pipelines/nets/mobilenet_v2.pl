# MobileNet-v2 probe: inverted residuals, valid depthwise convs (T=99)
pipeline mobilenet_v2
buffer input dims 3x672x672 elem 4
buffer conv1_w dims 32x3x3x3 elem 4
buffer dw3_w dims 32x3x3 elem 4
buffer project5_w dims 16x32x1x1 elem 4
buffer expand6_w dims 96x16x1x1 elem 4
buffer dw8_w dims 96x3x3 elem 4
buffer project10_w dims 24x96x1x1 elem 4
buffer expand11_w dims 144x24x1x1 elem 4
buffer dw13_w dims 144x3x3 elem 4
buffer project15_w dims 24x144x1x1 elem 4
buffer expand17_w dims 144x24x1x1 elem 4
buffer dw19_w dims 144x3x3 elem 4
buffer project21_w dims 32x144x1x1 elem 4
buffer expand22_w dims 192x32x1x1 elem 4
buffer dw24_w dims 192x3x3 elem 4
buffer project26_w dims 32x192x1x1 elem 4
buffer expand28_w dims 192x32x1x1 elem 4
buffer dw30_w dims 192x3x3 elem 4
buffer project32_w dims 32x192x1x1 elem 4
buffer expand34_w dims 192x32x1x1 elem 4
buffer dw36_w dims 192x3x3 elem 4
buffer project38_w dims 64x192x1x1 elem 4
buffer expand39_w dims 384x64x1x1 elem 4
buffer dw41_w dims 384x3x3 elem 4
buffer project43_w dims 64x384x1x1 elem 4
buffer expand45_w dims 384x64x1x1 elem 4
buffer dw47_w dims 384x3x3 elem 4
buffer project49_w dims 64x384x1x1 elem 4
buffer expand51_w dims 384x64x1x1 elem 4
buffer dw53_w dims 384x3x3 elem 4
buffer project55_w dims 64x384x1x1 elem 4
buffer expand57_w dims 384x64x1x1 elem 4
buffer dw59_w dims 384x3x3 elem 4
buffer project61_w dims 96x384x1x1 elem 4
buffer expand62_w dims 576x96x1x1 elem 4
buffer dw64_w dims 576x3x3 elem 4
buffer project66_w dims 96x576x1x1 elem 4
buffer expand68_w dims 576x96x1x1 elem 4
buffer dw70_w dims 576x3x3 elem 4
buffer project72_w dims 96x576x1x1 elem 4
buffer expand74_w dims 576x96x1x1 elem 4
buffer dw76_w dims 576x3x3 elem 4
buffer project78_w dims 160x576x1x1 elem 4
buffer expand79_w dims 960x160x1x1 elem 4
buffer dw81_w dims 960x3x3 elem 4
buffer project83_w dims 160x960x1x1 elem 4
buffer expand85_w dims 960x160x1x1 elem 4
buffer dw87_w dims 960x3x3 elem 4
buffer project89_w dims 160x960x1x1 elem 4
buffer expand91_w dims 960x160x1x1 elem 4
buffer dw93_w dims 960x3x3 elem 4
buffer project95_w dims 320x960x1x1 elem 4
buffer conv96_w dims 1280x320x1x1 elem 4
buffer fc99_w dims 1000x1280 elem 4
stage conv1 dims co:32,y:335,x:335 reduce ci:3 flops 18
  in input map ci*1+1, y*2+3, x*2+3
  in conv1_w map co*1+1, ci*1+1, _*0+3, _*0+3
stage relu2 dims c:32,y:335,x:335 flops 1
  in conv1 map c*1+1, y*1+1, x*1+1
stage dw3 dims c:32,y:333,x:333 flops 18
  in relu2 map c*1+1, y*1+3, x*1+3
  in dw3_w map c*1+1, _*0+3, _*0+3
stage relu4 dims c:32,y:333,x:333 flops 1
  in dw3 map c*1+1, y*1+1, x*1+1
stage project5 dims co:16,y:333,x:333 reduce ci:32 flops 2
  in relu4 map ci*1+1, y*1+1, x*1+1
  in project5_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage expand6 dims co:96,y:333,x:333 reduce ci:16 flops 2
  in project5 map ci*1+1, y*1+1, x*1+1
  in expand6_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu7 dims c:96,y:333,x:333 flops 1
  in expand6 map c*1+1, y*1+1, x*1+1
stage dw8 dims c:96,y:166,x:166 flops 18
  in relu7 map c*1+1, y*2+3, x*2+3
  in dw8_w map c*1+1, _*0+3, _*0+3
stage relu9 dims c:96,y:166,x:166 flops 1
  in dw8 map c*1+1, y*1+1, x*1+1
stage project10 dims co:24,y:166,x:166 reduce ci:96 flops 2
  in relu9 map ci*1+1, y*1+1, x*1+1
  in project10_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage expand11 dims co:144,y:166,x:166 reduce ci:24 flops 2
  in project10 map ci*1+1, y*1+1, x*1+1
  in expand11_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu12 dims c:144,y:166,x:166 flops 1
  in expand11 map c*1+1, y*1+1, x*1+1
stage dw13 dims c:144,y:164,x:164 flops 18
  in relu12 map c*1+1, y*1+3, x*1+3
  in dw13_w map c*1+1, _*0+3, _*0+3
stage relu14 dims c:144,y:164,x:164 flops 1
  in dw13 map c*1+1, y*1+1, x*1+1
stage project15 dims co:24,y:164,x:164 reduce ci:144 flops 2
  in relu14 map ci*1+1, y*1+1, x*1+1
  in project15_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add16 dims c:24,y:164,x:164 flops 1
  in project15 map c*1+1, y*1+1, x*1+1
  in project10 map c*1+1, y*1+1, x*1+1
stage expand17 dims co:144,y:164,x:164 reduce ci:24 flops 2
  in add16 map ci*1+1, y*1+1, x*1+1
  in expand17_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu18 dims c:144,y:164,x:164 flops 1
  in expand17 map c*1+1, y*1+1, x*1+1
stage dw19 dims c:144,y:81,x:81 flops 18
  in relu18 map c*1+1, y*2+3, x*2+3
  in dw19_w map c*1+1, _*0+3, _*0+3
stage relu20 dims c:144,y:81,x:81 flops 1
  in dw19 map c*1+1, y*1+1, x*1+1
stage project21 dims co:32,y:81,x:81 reduce ci:144 flops 2
  in relu20 map ci*1+1, y*1+1, x*1+1
  in project21_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage expand22 dims co:192,y:81,x:81 reduce ci:32 flops 2
  in project21 map ci*1+1, y*1+1, x*1+1
  in expand22_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu23 dims c:192,y:81,x:81 flops 1
  in expand22 map c*1+1, y*1+1, x*1+1
stage dw24 dims c:192,y:79,x:79 flops 18
  in relu23 map c*1+1, y*1+3, x*1+3
  in dw24_w map c*1+1, _*0+3, _*0+3
stage relu25 dims c:192,y:79,x:79 flops 1
  in dw24 map c*1+1, y*1+1, x*1+1
stage project26 dims co:32,y:79,x:79 reduce ci:192 flops 2
  in relu25 map ci*1+1, y*1+1, x*1+1
  in project26_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add27 dims c:32,y:79,x:79 flops 1
  in project26 map c*1+1, y*1+1, x*1+1
  in project21 map c*1+1, y*1+1, x*1+1
stage expand28 dims co:192,y:79,x:79 reduce ci:32 flops 2
  in add27 map ci*1+1, y*1+1, x*1+1
  in expand28_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu29 dims c:192,y:79,x:79 flops 1
  in expand28 map c*1+1, y*1+1, x*1+1
stage dw30 dims c:192,y:77,x:77 flops 18
  in relu29 map c*1+1, y*1+3, x*1+3
  in dw30_w map c*1+1, _*0+3, _*0+3
stage relu31 dims c:192,y:77,x:77 flops 1
  in dw30 map c*1+1, y*1+1, x*1+1
stage project32 dims co:32,y:77,x:77 reduce ci:192 flops 2
  in relu31 map ci*1+1, y*1+1, x*1+1
  in project32_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add33 dims c:32,y:77,x:77 flops 1
  in project32 map c*1+1, y*1+1, x*1+1
  in add27 map c*1+1, y*1+1, x*1+1
stage expand34 dims co:192,y:77,x:77 reduce ci:32 flops 2
  in add33 map ci*1+1, y*1+1, x*1+1
  in expand34_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu35 dims c:192,y:77,x:77 flops 1
  in expand34 map c*1+1, y*1+1, x*1+1
stage dw36 dims c:192,y:38,x:38 flops 18
  in relu35 map c*1+1, y*2+3, x*2+3
  in dw36_w map c*1+1, _*0+3, _*0+3
stage relu37 dims c:192,y:38,x:38 flops 1
  in dw36 map c*1+1, y*1+1, x*1+1
stage project38 dims co:64,y:38,x:38 reduce ci:192 flops 2
  in relu37 map ci*1+1, y*1+1, x*1+1
  in project38_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage expand39 dims co:384,y:38,x:38 reduce ci:64 flops 2
  in project38 map ci*1+1, y*1+1, x*1+1
  in expand39_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu40 dims c:384,y:38,x:38 flops 1
  in expand39 map c*1+1, y*1+1, x*1+1
stage dw41 dims c:384,y:36,x:36 flops 18
  in relu40 map c*1+1, y*1+3, x*1+3
  in dw41_w map c*1+1, _*0+3, _*0+3
stage relu42 dims c:384,y:36,x:36 flops 1
  in dw41 map c*1+1, y*1+1, x*1+1
stage project43 dims co:64,y:36,x:36 reduce ci:384 flops 2
  in relu42 map ci*1+1, y*1+1, x*1+1
  in project43_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add44 dims c:64,y:36,x:36 flops 1
  in project43 map c*1+1, y*1+1, x*1+1
  in project38 map c*1+1, y*1+1, x*1+1
stage expand45 dims co:384,y:36,x:36 reduce ci:64 flops 2
  in add44 map ci*1+1, y*1+1, x*1+1
  in expand45_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu46 dims c:384,y:36,x:36 flops 1
  in expand45 map c*1+1, y*1+1, x*1+1
stage dw47 dims c:384,y:34,x:34 flops 18
  in relu46 map c*1+1, y*1+3, x*1+3
  in dw47_w map c*1+1, _*0+3, _*0+3
stage relu48 dims c:384,y:34,x:34 flops 1
  in dw47 map c*1+1, y*1+1, x*1+1
stage project49 dims co:64,y:34,x:34 reduce ci:384 flops 2
  in relu48 map ci*1+1, y*1+1, x*1+1
  in project49_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add50 dims c:64,y:34,x:34 flops 1
  in project49 map c*1+1, y*1+1, x*1+1
  in add44 map c*1+1, y*1+1, x*1+1
stage expand51 dims co:384,y:34,x:34 reduce ci:64 flops 2
  in add50 map ci*1+1, y*1+1, x*1+1
  in expand51_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu52 dims c:384,y:34,x:34 flops 1
  in expand51 map c*1+1, y*1+1, x*1+1
stage dw53 dims c:384,y:32,x:32 flops 18
  in relu52 map c*1+1, y*1+3, x*1+3
  in dw53_w map c*1+1, _*0+3, _*0+3
stage relu54 dims c:384,y:32,x:32 flops 1
  in dw53 map c*1+1, y*1+1, x*1+1
stage project55 dims co:64,y:32,x:32 reduce ci:384 flops 2
  in relu54 map ci*1+1, y*1+1, x*1+1
  in project55_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add56 dims c:64,y:32,x:32 flops 1
  in project55 map c*1+1, y*1+1, x*1+1
  in add50 map c*1+1, y*1+1, x*1+1
stage expand57 dims co:384,y:32,x:32 reduce ci:64 flops 2
  in add56 map ci*1+1, y*1+1, x*1+1
  in expand57_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu58 dims c:384,y:32,x:32 flops 1
  in expand57 map c*1+1, y*1+1, x*1+1
stage dw59 dims c:384,y:30,x:30 flops 18
  in relu58 map c*1+1, y*1+3, x*1+3
  in dw59_w map c*1+1, _*0+3, _*0+3
stage relu60 dims c:384,y:30,x:30 flops 1
  in dw59 map c*1+1, y*1+1, x*1+1
stage project61 dims co:96,y:30,x:30 reduce ci:384 flops 2
  in relu60 map ci*1+1, y*1+1, x*1+1
  in project61_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage expand62 dims co:576,y:30,x:30 reduce ci:96 flops 2
  in project61 map ci*1+1, y*1+1, x*1+1
  in expand62_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu63 dims c:576,y:30,x:30 flops 1
  in expand62 map c*1+1, y*1+1, x*1+1
stage dw64 dims c:576,y:28,x:28 flops 18
  in relu63 map c*1+1, y*1+3, x*1+3
  in dw64_w map c*1+1, _*0+3, _*0+3
stage relu65 dims c:576,y:28,x:28 flops 1
  in dw64 map c*1+1, y*1+1, x*1+1
stage project66 dims co:96,y:28,x:28 reduce ci:576 flops 2
  in relu65 map ci*1+1, y*1+1, x*1+1
  in project66_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add67 dims c:96,y:28,x:28 flops 1
  in project66 map c*1+1, y*1+1, x*1+1
  in project61 map c*1+1, y*1+1, x*1+1
stage expand68 dims co:576,y:28,x:28 reduce ci:96 flops 2
  in add67 map ci*1+1, y*1+1, x*1+1
  in expand68_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu69 dims c:576,y:28,x:28 flops 1
  in expand68 map c*1+1, y*1+1, x*1+1
stage dw70 dims c:576,y:26,x:26 flops 18
  in relu69 map c*1+1, y*1+3, x*1+3
  in dw70_w map c*1+1, _*0+3, _*0+3
stage relu71 dims c:576,y:26,x:26 flops 1
  in dw70 map c*1+1, y*1+1, x*1+1
stage project72 dims co:96,y:26,x:26 reduce ci:576 flops 2
  in relu71 map ci*1+1, y*1+1, x*1+1
  in project72_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add73 dims c:96,y:26,x:26 flops 1
  in project72 map c*1+1, y*1+1, x*1+1
  in add67 map c*1+1, y*1+1, x*1+1
stage expand74 dims co:576,y:26,x:26 reduce ci:96 flops 2
  in add73 map ci*1+1, y*1+1, x*1+1
  in expand74_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu75 dims c:576,y:26,x:26 flops 1
  in expand74 map c*1+1, y*1+1, x*1+1
stage dw76 dims c:576,y:12,x:12 flops 18
  in relu75 map c*1+1, y*2+3, x*2+3
  in dw76_w map c*1+1, _*0+3, _*0+3
stage relu77 dims c:576,y:12,x:12 flops 1
  in dw76 map c*1+1, y*1+1, x*1+1
stage project78 dims co:160,y:12,x:12 reduce ci:576 flops 2
  in relu77 map ci*1+1, y*1+1, x*1+1
  in project78_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage expand79 dims co:960,y:12,x:12 reduce ci:160 flops 2
  in project78 map ci*1+1, y*1+1, x*1+1
  in expand79_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu80 dims c:960,y:12,x:12 flops 1
  in expand79 map c*1+1, y*1+1, x*1+1
stage dw81 dims c:960,y:10,x:10 flops 18
  in relu80 map c*1+1, y*1+3, x*1+3
  in dw81_w map c*1+1, _*0+3, _*0+3
stage relu82 dims c:960,y:10,x:10 flops 1
  in dw81 map c*1+1, y*1+1, x*1+1
stage project83 dims co:160,y:10,x:10 reduce ci:960 flops 2
  in relu82 map ci*1+1, y*1+1, x*1+1
  in project83_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add84 dims c:160,y:10,x:10 flops 1
  in project83 map c*1+1, y*1+1, x*1+1
  in project78 map c*1+1, y*1+1, x*1+1
stage expand85 dims co:960,y:10,x:10 reduce ci:160 flops 2
  in add84 map ci*1+1, y*1+1, x*1+1
  in expand85_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu86 dims c:960,y:10,x:10 flops 1
  in expand85 map c*1+1, y*1+1, x*1+1
stage dw87 dims c:960,y:8,x:8 flops 18
  in relu86 map c*1+1, y*1+3, x*1+3
  in dw87_w map c*1+1, _*0+3, _*0+3
stage relu88 dims c:960,y:8,x:8 flops 1
  in dw87 map c*1+1, y*1+1, x*1+1
stage project89 dims co:160,y:8,x:8 reduce ci:960 flops 2
  in relu88 map ci*1+1, y*1+1, x*1+1
  in project89_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage add90 dims c:160,y:8,x:8 flops 1
  in project89 map c*1+1, y*1+1, x*1+1
  in add84 map c*1+1, y*1+1, x*1+1
stage expand91 dims co:960,y:8,x:8 reduce ci:160 flops 2
  in add90 map ci*1+1, y*1+1, x*1+1
  in expand91_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu92 dims c:960,y:8,x:8 flops 1
  in expand91 map c*1+1, y*1+1, x*1+1
stage dw93 dims c:960,y:6,x:6 flops 18
  in relu92 map c*1+1, y*1+3, x*1+3
  in dw93_w map c*1+1, _*0+3, _*0+3
stage relu94 dims c:960,y:6,x:6 flops 1
  in dw93 map c*1+1, y*1+1, x*1+1
stage project95 dims co:320,y:6,x:6 reduce ci:960 flops 2
  in relu94 map ci*1+1, y*1+1, x*1+1
  in project95_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage conv96 dims co:1280,y:6,x:6 reduce ci:320 flops 2
  in project95 map ci*1+1, y*1+1, x*1+1
  in conv96_w map co*1+1, ci*1+1, _*0+1, _*0+1
stage relu97 dims c:1280,y:6,x:6 flops 1
  in conv96 map c*1+1, y*1+1, x*1+1
stage gap98 dims c:1280 reduce y:6,x:6 flops 1
  in relu97 map c*1+1, y*1+1, x*1+1
stage fc99 dims o:1000 reduce i:1280 flops 2 output
  in gap98 map i*1+1
  in fc99_w map o*1+1, i*1+1

// Host-side check of the 2-bit (labels, final) unpack used by ef_canny_u8_host:
// every length / output offset against a scalar decode (compiled and run by
// tests/test_cpu_host.py against the built library).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cstring>
namespace ef { void unpack_codes(const uint8_t*, size_t, size_t, size_t, uint8_t*, uint8_t*); }
int main(){
  for (size_t npx : {1ul, 3ul, 4ul, 5ul, 31ul, 32ul, 33ul, 127ul, 1000ul, 4099ul, 100003ul}) {
    for (int off : {0, 1, 4, 16, 32}) {
      size_t nb=(npx+3)/4; std::vector<uint8_t> p(nb+8); for (size_t i=0;i<nb;i++) p[i]=(uint8_t)(rand());
      std::vector<uint8_t> L(npx+64+off,7), F(npx+64+off,7);
      ef::unpack_codes(p.data(), 0, nb, npx, L.data()+off, F.data()+off);
      for (size_t i=0;i<npx;i++){int c=(p[i/4]>>(2*(i%4)))&3; int l=c==0?0:(c==3?2:1); int f=c>=2; if(L[off+i]!=l||F[off+i]!=f){printf("FAIL npx=%zu off=%d i=%zu\n",npx,off,i);return 1;}}
      if (L[off+npx]!=7||F[off+npx]!=7){printf("overrun\n");return 1;}
    }
  }
  printf("unpack ok\n"); return 0;
}

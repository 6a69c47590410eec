/* How much of the JP bulk is independent of the core prefix (no pred chain into
 * the core)?  Reads g.bin = {n, nnz, off[n+1], col[nnz], round[n]} (int64,
 * int64, int64[], int32[], int32[]); seed 1, core = first 65535 in priority
 * order.  R-MAT 24: 1.0 % of the bulk (all round 1), so the bulk cannot
 * usefully run beside the core. */
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
static uint64_t h(uint64_t seed, uint32_t v){uint64_t z=(seed^(uint64_t)v)+0x9E3779B97F4A7C15ull;z=(z^(z>>30))*0xBF58476D1CE4E5B9ull;z=(z^(z>>27))*0x94D049BB133111EBull;return z^(z>>31);}
int n; int64_t *off; int32_t *col,*rnd; int64_t *ord;
static int cmp(const void*a,const void*b){int64_t x=*(int64_t*)a,y=*(int64_t*)b; if(rnd[x]!=rnd[y]) return rnd[x]>rnd[y]?-1:1; uint64_t hx=h(1,x),hy=h(1,y); return hx>hy?-1:(hx<hy?1:0);}
int main(){FILE*f=fopen("g.bin","rb"); int64_t nn,nnz; fread(&nn,8,1,f);fread(&nnz,8,1,f); n=nn; off=malloc(8*(n+1)); col=malloc(4*nnz); rnd=malloc(4*n); fread(off,8,n+1,f); fread(col,4,nnz,f); fread(rnd,4,n,f); fclose(f);
 int64_t m=0; ord=malloc(8*n); for(int v=0;v<n;v++) if(off[v+1]>off[v]) ord[m++]=v;
 qsort(ord,m,8,cmp);
 int64_t *pos=malloc(8*n); for(int64_t i=0;i<m;i++) pos[ord[i]]=i;
 char*dep=calloc(n,1); int NC=65535;
 int64_t indep=0, indep_arcs=0, tot_arcs=0; int64_t firstdep_hist[10]={0};
 for(int64_t i=0;i<m;i++){int v=ord[i]; if(i<NC){dep[v]=1;continue;} int d=0; for(int64_t e=off[v];e<off[v+1];e++){int u=col[e]; if(pos[u]<i && dep[u]){d=1;break;}} dep[v]=d; if(!d){indep++;} }
 printf("n_order %ld core %d bulk %ld independent %ld (%.1f%%)\n",m,NC,m-NC,indep,100.0*indep/(m-NC));
 // by round
 for(int r=1;r<=7;r++){int64_t c=0,ci=0; for(int64_t i=NC;i<m;i++){int v=ord[i]; if(rnd[v]==r){c++; if(!dep[v]) ci++;}} printf("round %d bulk %ld indep %ld\n",r,c,ci);}
 return 0;}

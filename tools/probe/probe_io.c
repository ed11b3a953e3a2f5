// Storage probe: O_DIRECT / buffered sequential read bandwidth with T threads.
#define _GNU_SOURCE
#include <fcntl.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>
#include <stdint.h>
static double now(){struct timespec t;clock_gettime(CLOCK_MONOTONIC,&t);return t.tv_sec+t.tv_nsec*1e-9;}
typedef struct{const char*path;int direct;size_t req;off_t lo,hi;int qd;}arg_t;
static void* worker(void*p){arg_t*a=p;int fd=open(a->path,O_RDONLY|(a->direct?O_DIRECT:0));if(fd<0){perror("open");return 0;}
 void*buf;posix_memalign(&buf,4096,a->req);for(off_t o=a->lo;o<a->hi;o+=a->req){ssize_t n=pread(fd,buf,a->req,o);if(n<=0){perror("pread");break;}}
 free(buf);close(fd);return 0;}
static void* writer(void*p){arg_t*a=p;int fd=open(a->path,O_WRONLY);void*buf;posix_memalign(&buf,4096,a->req);
 for(off_t o=a->lo;o<a->hi;o+=a->req){uint64_t*w=buf;for(size_t i=0;i<a->req/8;i++)w[i]=(o/8+i)*0x9E3779B97F4A7C15ull;pwrite(fd,buf,a->req,o);}free(buf);close(fd);return 0;}
int main(int argc,char**argv){const char*path=argv[1];size_t size=strtoull(argv[2],0,0)<<20;
 if(argc>3&&!strcmp(argv[3],"create")){int fd=open(path,O_CREAT|O_WRONLY|O_TRUNC,0644);ftruncate(fd,size);close(fd);
  int T=16;pthread_t th[64];arg_t a[64];double t0=now();for(int i=0;i<T;i++){a[i]=(arg_t){path,0,1<<20,size/T*i,size/T*(i+1)};pthread_create(&th[i],0,writer,&a[i]);}
  for(int i=0;i<T;i++)pthread_join(th[i],0);int fd2=open(path,O_WRONLY);fsync(fd2);close(fd2);printf("create %zu MiB: %.2f GB/s\n",size>>20,size/(now()-t0)/1e9);return 0;}
 int threads[]={1,2,4,8,16,32};size_t reqs[]={65536,1<<20,4<<20,16<<20};
 for(int d=1;d>=0;d--)for(int ri=0;ri<4;ri++)for(int ti=0;ti<6;ti++){int T=threads[ti];size_t req=reqs[ri];pthread_t th[64];arg_t a[64];
  if(T>sysconf(_SC_NPROCESSORS_ONLN)*2)continue;
  double t0=now();for(int i=0;i<T;i++){a[i]=(arg_t){path,d,req,size/T*i,size/T*(i+1)};pthread_create(&th[i],0,worker,&a[i]);}
  for(int i=0;i<T;i++)pthread_join(th[i],0);double dt=now()-t0;printf("%s req=%zuK threads=%d: %.2f GB/s\n",d?"ODIRECT":"buffered",req>>10,T,size/dt/1e9);fflush(stdout);}
 return 0;}

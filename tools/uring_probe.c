#include <linux/io_uring.h>
#include <sys/syscall.h>
#include <unistd.h>
#include <stdio.h>
#include <string.h>
#include <errno.h>
int main(){ struct io_uring_params p; memset(&p,0,sizeof p); int fd=syscall(__NR_io_uring_setup, 8, &p); printf("io_uring_setup -> %d errno=%d (%s) features=0x%x\n", fd, fd<0?errno:0, fd<0?strerror(errno):"", p.features); return 0;}

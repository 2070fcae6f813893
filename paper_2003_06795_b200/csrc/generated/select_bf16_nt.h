#ifndef SELECT_BF16_NT_H
#define SELECT_BF16_NT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_nt_config;

static inline select_bf16_nt_config select_bf16_nt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(3584)) {
        if (n < INT64_C(444)) {
            if (n < INT64_C(287)) {
                if (n < INT64_C(222)) {
                    if (k < INT64_C(744)) {
                        if (m < INT64_C(159)) {
                            if (m < INT64_C(57)) {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(28)) {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(46)) {
                                    if (k < INT64_C(167)) {
                                        if (m < INT64_C(2218)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(111)) {
                                        if (m < INT64_C(2218)) {
                                            if (m < INT64_C(278)) {
                                                if (k < INT64_C(471)) {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(471)) {
                                                    if (n < INT64_C(79)) {
                                                        if (m < INT64_C(555)) {
                                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(471)) {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(2218)) {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(725)) {
                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(555)) {
                            if (m < INT64_C(278)) {
                                if (k < INT64_C(1536)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(2218)) {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(1087)) {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(1630)) {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(2218)) {
                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            }
        } else {
            if (m < INT64_C(2218)) {
                if (k < INT64_C(1620)) {
                    if (m < INT64_C(448)) {
                        if (k < INT64_C(124)) {
                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(1012)) {
                                if (m < INT64_C(70)) {
                                    if (m < INT64_C(12)) {
                                        if (m < INT64_C(2)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(139)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(287)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(725)) {
                                            if (m < INT64_C(139)) {
                                                if (m < INT64_C(70)) {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (m < INT64_C(70)) {
                                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(139)) {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(744)) {
                            if (m < INT64_C(634)) {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(111)) {
                                    if (m < INT64_C(1109)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(405)) {
                                if (m < INT64_C(1109)) {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(896)) {
                                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(1268)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(6)) {
                        if (n < INT64_C(2024)) {
                            if (m < INT64_C(3)) {
                                if (m < INT64_C(2)) {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(2897)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(2897)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (m < INT64_C(12)) {
                                if (k < INT64_C(2897)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(10138)) {
                                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(1109)) {
                                    if (k < INT64_C(2173)) {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(3259)) {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                return out;
            }
        }
    } else {
        if (k < INT64_C(815)) {
            if (m < INT64_C(17740)) {
                if (n < INT64_C(91)) {
                    if (k < INT64_C(42)) {
                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(118)) {
                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(192)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(384)) {
                                        select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(46)) {
                                    select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(194)) {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(384)) {
                                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(8870)) {
                        if (k < INT64_C(46)) {
                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(363)) {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(111)) {
                    if (m < INT64_C(35480)) {
                        if (n < INT64_C(46)) {
                            select_bf16_nt_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(70960)) {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (n < INT64_C(363)) {
                if (m < INT64_C(35480)) {
                    if (m < INT64_C(8870)) {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(17740)) {
                            if (k < INT64_C(1630)) {
                                if (n < INT64_C(182)) {
                                    select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                select_bf16_nt_config out = {8u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_NT_H */
